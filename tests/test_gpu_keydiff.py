"""K6 KeyDiff baseline scorer (keydiff_scores, scoring.hpp:186-221) on the GPU
vs the oracle restatement (itself pinned bit for bit to the reference by
test_oracle_vs_ref.py / test_golden.py): fp64 scores bit-exact for bf16, fp32
and fp64 caches (ragged heads with slack gaps, an empty head, zero keys, a
zero-anchor head), the retained sets of the shared select + compaction path
bit-exact with evict_to_budget, and a chained KeyDiff block prefill."""
import numpy as np
import pytest
import torch

from tests.helpers import bf16_round, random_layer

pytestmark = pytest.mark.gpu

TORCH = {"bf16": torch.bfloat16, "f32": torch.float32, "f64": torch.float64}


def _cache(gpu, rng, L, H, d, counts_per_layer, dtype, slack=3, zero_key=False, zero_head=False):
    layers = []
    for l in range(L):
        ho, pos, k, v = random_layer(rng, H, counts_per_layer[l], d)
        if dtype == "bf16":
            k, v = bf16_round(k), bf16_round(v)
        elif dtype == "f32":
            k, v = k.astype(np.float32).astype(np.float64), v.astype(np.float32).astype(np.float64)
        if zero_key and len(pos):
            k[rng.integers(0, len(pos), 3)] = 0.0
        if zero_head and ho[1] > ho[0]:
            k[ho[0]:ho[1]] = 0.0
        layers.append((ho, pos, k, v))
    cap = [int(ho[-1]) + slack * H for ho, _, _, _ in layers]
    c = gpu.EpisodeCache(L, H, d, cap, TORCH[dtype], "cuda")
    c.load_layers([(np.diff(ho), pos, k, v) for ho, pos, k, v in layers])
    return layers, c


@pytest.mark.parametrize("dtype", ["bf16", "f32", "f64"])
def test_keydiff_scores_bitexact(gpu, orc, dtype):
    rng = np.random.default_rng({"bf16": 1, "f32": 2, "f64": 3}[dtype])
    L, H, d = 3, 4, 128
    counts = [[300, 0, 129, 77], [1, 2, 3, 500], [256, 256, 256, 256]]
    layers, c = _cache(gpu, rng, L, H, d, counts, dtype, zero_key=True, zero_head=(dtype == "f32"))
    sc = gpu.keydiff_scores(c).cpu().numpy()
    for l, (ho, pos, k, _) in enumerate(layers):
        exp = orc.keydiff_layer(k, ho)
        got = sc[c.live_rows(l).cpu().numpy()]
        assert np.array_equal(got, exp), (dtype, l)


def test_keydiff_small_head_dim_and_single_row(gpu, orc):
    rng = np.random.default_rng(9)
    for d, counts in [(4, [[1, 7]]), (64, [[33, 0, 2]]), (256, [[40]])]:
        H = len(counts[0])
        layers, c = _cache(gpu, rng, 1, H, d, counts, "f64")
        sc = gpu.keydiff_scores(c).cpu().numpy()
        ho, pos, k, _ = layers[0]
        got = sc[c.live_rows(0).cpu().numpy()]
        assert np.array_equal(got, orc.keydiff_layer(k, ho)), d


def test_keydiff_select_compact_matches_evict_to_budget(gpu, orc):
    """KeyDiff scores -> pooled select -> compaction == evict_to_budget on the
    same scores (retained positions and K/V rows)."""
    rng = np.random.default_rng(4)
    L, H, d = 2, 8, 128
    counts = [[1280] * H, [900, 1500, 0, 77, 1280, 2000, 640, 129]]
    budgets = [1024, 400]
    layers, c = _cache(gpu, rng, L, H, d, counts, "bf16", slack=64)
    sc = gpu.keydiff_scores(c)
    keep = gpu.select_pooled(c, sc, budgets)
    out = gpu.EpisodeCache(L, H, d, [int(ho[-1]) + 64 * H for ho, _, _, _ in layers], torch.bfloat16, "cuda")
    gpu.compact(c, keep, out, slack=64)
    torch.cuda.synchronize()
    got = out.retained_positions()
    for l, (ho, pos, k, _) in enumerate(layers):
        st, kp = orc.evict_layer(ho, pos, orc.keydiff_layer(k, ho), budgets[l])
        assert st >= 0
        ref = [pos[ho[h]:ho[h + 1]][kp[ho[h]:ho[h + 1]]].tolist() for h in range(H)]
        assert got[l] == ref, l


def test_keydiff_block_prefill_chain(gpu, orc):
    """block_prefill(scorer="keydiff") vs the oracle chained block by block."""
    from tests.test_gpu_blockprefill import SynthProvider
    L, Hq, H, d, n, B, M = 2, 4, 2, 16, 96, 16, 8
    prov = SynthProvider(L, Hq, H, d, n, 3, seed=5, dtype=torch.float32)
    cfg = gpu.BlockPrefillConfig(M, B, scorer="keydiff")
    rep = gpu.block_prefill(prov, L, Hq, H, d, n, cfg, dtype=torch.float32)
    # oracle: per layer, per head lists of (position, key)
    kf = prov.k.double().numpy()
    state = [[[] for _ in range(H)] for _ in range(L)]
    for start in range(0, n, B):
        for l in range(L):
            for h in range(H):
                state[l][h] += list(range(start, min(n, start + B)))
            ho = np.concatenate([[0], np.cumsum([len(s) for s in state[l]])])
            pos = np.concatenate([np.array(s, np.int64) for s in state[l]])
            k = np.concatenate([kf[l, h, state[l][h]] for h in range(H)])
            st, keep = orc.evict_layer(ho, pos, orc.keydiff_layer(k, ho), M)
            assert st >= 0
            state[l] = [pos[ho[h]:ho[h + 1]][keep[ho[h]:ho[h + 1]]].tolist() for h in range(H)]
    assert rep.cache.retained_positions() == state
