"""K7 episodic cache store on the GPU: the device writer (epk_serialize_epkv)
produces the reference's persist bytes exactly (bf16 / fp32 / fp64 caches,
ragged and empty heads, caches with slack gaps straight out of block
prefill), the reference reads our files back, load_cache + persist round-trip
byte for byte, and the CacheStore / route load-on-switch rule."""
import os

import numpy as np
import pytest
import torch

from tests.helpers import bf16_round, random_layer

pytestmark = pytest.mark.gpu

TORCH = {"bf16": torch.bfloat16, "f32": torch.float32, "f64": torch.float64}


def _data(rng, L, H, d, counts, dtype):
    pl = []
    for l in range(L):
        ho, pos, k, v = random_layer(rng, H, counts[l], d)
        if dtype == "bf16":
            k, v = bf16_round(k), bf16_round(v)
        elif dtype == "f32":
            k, v = k.astype(np.float32).astype(np.float64), v.astype(np.float32).astype(np.float64)
        pl.append((np.diff(ho), pos.astype(np.int64), k, v))
    return pl


@pytest.mark.parametrize("dtype", ["bf16", "f32", "f64"])
def test_persist_bytes_equal_reference(gpu, ref, tmp_path, dtype):
    rng = np.random.default_rng({"bf16": 1, "f32": 2, "f64": 3}[dtype])
    L, H, d = 3, 4, 128 if dtype != "f64" else 16
    pl = _data(rng, L, H, d, [[30, 0, 7, 12], [1, 1, 1, 1], [0, 0, 0, 5]], dtype)
    cache = gpu.EpisodeCache(L, H, d, [int(c.sum()) + 8 * H for c, _, _, _ in pl], TORCH[dtype], "cuda")
    cache.load_layers(pl, slack=8)  # gaps between heads: the writer must skip them
    budgets = [10, 20, 30]
    ours = tmp_path / "ours.epkv"
    n = gpu.persist(cache, ours, episode_id=11, scorer="patched", budget_per_head=20, layer_budgets=budgets)
    theirs = tmp_path / "ref.epkv"
    m = ref.ref_persist(theirs, pl, episode_id=11, scorer="patched", budget_per_head=20, layer_budgets=budgets,
                        layer_budget_fields=budgets)
    assert n == m and ours.read_bytes() == theirs.read_bytes()
    # the reference reads our file (load_cache -> persist reproduces it)
    again = tmp_path / "again.epkv"
    assert ref.ref_load_repersist(ours, again) == n and again.read_bytes() == ours.read_bytes()


def test_load_and_round_trip(gpu, ref, tmp_path):
    rng = np.random.default_rng(7)
    pl = _data(rng, 2, 8, 128, [[100] * 8, [3, 0, 50, 7, 1, 0, 2, 9]], "bf16")
    src = tmp_path / "src.epkv"
    ref.ref_persist(src, pl, episode_id=2, scorer="keydiff", budget_per_head=64, layer_budgets=[64, 64],
                    layer_budget_fields=[64, 64])
    cache, meta = gpu.load_cache(src, dtype=torch.bfloat16, slack=16)
    assert (meta.episode_id, meta.scorer, meta.budget_per_head) == (2, "keydiff", 64)
    for l, (c, p, k, v) in enumerate(pl):
        ln, pos, kk, vv = cache.layer_view(l)
        assert np.array_equal(ln, c) and np.array_equal(pos, p)
        assert np.array_equal(kk.double().numpy(), k) and np.array_equal(vv.double().numpy(), v)
    out = tmp_path / "out.epkv"
    gpu.persist(cache, out, episode_id=2, scorer="keydiff", budget_per_head=64, layer_budgets=[64, 64])
    assert out.read_bytes() == src.read_bytes()
    with pytest.raises(gpu.Error, match="not exactly representable"):
        pl64 = _data(rng, 1, 1, 4, [[3]], "f64")
        ref.ref_persist(tmp_path / "x.epkv", pl64, budget_per_head=1)
        gpu.load_cache(tmp_path / "x.epkv", dtype=torch.bfloat16)


def test_block_prefill_cache_persists_like_reference(gpu, ref, tmp_path):
    """A cache straight out of the GPU block prefill (ragged heads, slack) persists
    to the bytes the reference writes for the same retained entries."""
    from tests.test_gpu_blockprefill import SynthProvider
    prov = SynthProvider(2, 4, 2, 16, 96, 3, seed=2, dtype=torch.float32)
    rep = gpu.block_prefill(prov, 2, 4, 2, 16, 96, gpu.BlockPrefillConfig(8, 16, scorer="keydiff"),
                            dtype=torch.float32)
    ours = tmp_path / "bp.epkv"
    gpu.persist(rep.cache, ours, episode_id=0, scorer="keydiff", budget_per_head=8, layer_budgets=rep.layer_budgets)
    pl = [tuple(x if not torch.is_tensor(x) else x.double().numpy() for x in rep.cache.layer_view(l))
          for l in range(2)]
    theirs = tmp_path / "bp_ref.epkv"
    ref.ref_persist(theirs, pl, scorer="keydiff", budget_per_head=8, layer_budgets=rep.layer_budgets,
                    layer_budget_fields=rep.layer_budgets)
    assert ours.read_bytes() == theirs.read_bytes()


def test_cache_store_and_route(gpu, tmp_path):
    rng = np.random.default_rng(9)
    st = gpu.CacheStore(tmp_path / "store")
    centroids = [rng.standard_normal(32) for _ in range(3)]
    for e in range(3):
        pl = _data(rng, 1, 2, 8, [[4 + e, 2]], "bf16")
        c = gpu.EpisodeCache(1, 2, 8, [int(pl[0][0].sum())], torch.bfloat16, "cuda")
        c.load_layers(pl)
        n = st.save(c, e, scorer="patched", budget_per_head=4, layer_budgets=[4])
        assert n == st.stored_bytes(e) > 0
    man = gpu.manifest_json(centroids, [(0, 1)] * 3, ["a", "b", "c"], st, "patched", 4, [4], 32)
    st.write_manifest(man)
    assert st.read_manifest() == man
    assert list(man) == ["version", "embedder_dim", "budget_per_head", "scorer", "layer_budgets", "episodes"]
    state = gpu.SessionState()
    seq = [centroids[1] * 2, centroids[1] + 1e-3, centroids[0], centroids[2], centroids[2]]
    got = [gpu.route(st, centroids, q, state) for q in seq]
    assert got == [1, 1, 0, 2, 2]
    assert state.switch_count == 3 and [r.switched for r in state.route_log] == [True, False, True, True, False]
    assert state.resident.entries_per_layer() == [4 + 2 + 2]
    with pytest.raises(gpu.IoError, match="unknown episode id"):
        st.load(9)


@pytest.mark.parametrize("dtype", ["bf16", "f32", "f64"])
def test_device_retrieve_equals_host_load(gpu, tmp_path, dtype):
    """Phase B retrieve on the GPU (epk_epkv_scan + epk_load_epkv): the same
    cache, positions, metadata and per-layer budget fields as the host
    load_cache; values that do not round-trip to the dtype fail closed; a
    truncated file fails closed."""
    rng = np.random.default_rng({"bf16": 4, "f32": 5, "f64": 6}[dtype])
    L, H, d = 3, 4, 128 if dtype != "f64" else 16
    pl = _data(rng, L, H, d, [[30, 0, 7, 12], [1, 1, 1, 1], [0, 0, 0, 5]], dtype)
    cache = gpu.EpisodeCache(L, H, d, [int(c.sum()) + 8 * H for c, _, _, _ in pl], TORCH[dtype], "cuda")
    cache.load_layers(pl, slack=8)
    src = tmp_path / "c.epkv"
    gpu.persist(cache, src, episode_id=5, scorer="patched", budget_per_head=9, layer_budgets=[3, 4, 5])
    a, ma = gpu.load_cache(src, dtype=TORCH[dtype], slack=4)
    b, mb = gpu.retrieve(src, dtype=TORCH[dtype], slack=4)
    assert ma == mb
    assert torch.equal(a.head_off, b.head_off) and torch.equal(a.head_len, b.head_len)
    for l in range(L):
        ra, rb = a.live_rows(l), b.live_rows(l)
        assert torch.equal(a.pos[ra], b.pos[rb])
        assert torch.equal(a.k[ra].view(torch.uint8), b.k[rb].view(torch.uint8))
        assert torch.equal(a.v[ra].view(torch.uint8), b.v[rb].view(torch.uint8))
    if dtype == "f64":  # fp64 values do not fit bf16: fail closed like load_cache(exact=True)
        with pytest.raises(gpu.Error):
            gpu.retrieve(src, dtype=torch.bfloat16)
    cut = tmp_path / "cut.epkv"
    cut.write_bytes(src.read_bytes()[:-7])
    with pytest.raises(gpu.IoError):
        gpu.retrieve(cut)
