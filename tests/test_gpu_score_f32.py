"""K1' (fp32 parity scorer) vs the oracle: bit-exact against the EPK-F32 v1
restatement, within 1e-5 relative of the reference fp64 scores, and
retained sets / compacted layout bit-exact after selection.  Also the
drop-in grid scorer (score_with_prompt on given grids) bit-exact vs fp64."""
import os

import numpy as np
import pytest
import torch

from tests.helpers import bf16_round, random_layer

pytestmark = pytest.mark.gpu


def _cache_from_layers(epk, layers, d, dtype, slack=0):
    H = len(layers[0][0]) - 1
    cap = [int(ho[-1]) + slack * H + 1 for ho, _, _, _ in layers]
    c = epk.EpisodeCache(len(layers), H, d, cap, dtype, "cuda")
    c.load_layers([(np.diff(ho), pos, k, v) for ho, pos, k, v in layers])
    return c


def test_expf_bitwise(gpu, orc):
    from paper_2509_17396_b200.scoring import debug_expf
    x = np.concatenate([np.linspace(-110, 1, 2_000_001), -np.abs(np.random.default_rng(0).standard_normal(100000)) * 30])
    x = x.astype(np.float32)
    y = debug_expf(torch.as_tensor(x, device="cuda")).cpu().numpy()
    assert np.array_equal(y.view(np.uint32), orc.expf(x).view(np.uint32))


@pytest.mark.parametrize("agg", ["max", "avg"])
@pytest.mark.parametrize("shape", [(6, 2, 16, 5, [13, 9]), (24, 8, 128, 64, [257] * 8), (4, 4, 32, 1, [0, 30, 1, 70]),
                                   (28, 4, 128, 17, [600, 513, 9, 1000])])
def test_exact_f32_bitwise_vs_oracle(gpu, orc, agg, shape):
    hq, H, d, p, counts = shape
    rng = np.random.default_rng(sum(counts) + p)
    L = 2
    layers, qs, kps = [], [], []
    for _ in range(L):
        ho, pos, k, v = random_layer(rng, H, counts, d, dtype=np.float32)
        layers.append((ho, pos, k, v))
        qs.append(rng.standard_normal((hq, p, d)).astype(np.float32))
        kps.append(rng.standard_normal((H, p, d)).astype(np.float32))
    c = _cache_from_layers(gpu, layers, d, torch.float32)
    q = torch.as_tensor(np.stack(qs), device="cuda")
    kp = torch.as_tensor(np.stack(kps), device="cuda")
    sc = gpu.score_with_prompt(c, q, kp, agg, mode="exact_f32").cpu().numpy()
    for l, (ho, pos, k, v) in enumerate(layers):
        exp = orc.score_layer_f32(qs[l], k, kps[l], ho, agg == "max")
        b = int(c.layer_base[l])
        got = sc[b:b + len(pos)]
        assert np.array_equal(got.view(np.uint32), exp.view(np.uint32)), (l, np.abs(got - exp).max())


def test_exact_f32_vs_fp64_reference_1e5(gpu, orc):
    """north_star: scores within 1e-5 relative of the fp64 reference path."""
    rng = np.random.default_rng(77)
    hq, H, d, p = 24, 8, 128, 64
    ho, pos, k, v = random_layer(rng, H, [1500] * H, d, dtype=np.float32)
    k = bf16_round(k)
    q = bf16_round(rng.standard_normal((hq, p, d)).astype(np.float32))
    kp = bf16_round(rng.standard_normal((H, p, d)).astype(np.float32))
    c = _cache_from_layers(gpu, [(ho, pos, k, v)], d, torch.float32)
    sc = gpu.score_with_prompt(c, torch.as_tensor(q[None], device="cuda"), torch.as_tensor(kp[None], device="cuda"),
                               "max", mode="exact_f32").cpu().numpy()[: len(pos)]
    ref64 = orc.score_layer_f64(q.astype(np.float64), k.astype(np.float64), kp.astype(np.float64), ho, True)
    rel = np.abs(sc.astype(np.float64) - ref64) / ref64
    assert rel.max() < 1e-5, rel.max()


def test_retained_sets_and_layout_bitexact_fp32_path(gpu, orc):
    """score (fp32) -> pooled select -> compact equals the oracle chain
    bit for bit: retained sets, per-head counts, compacted K/V/positions."""
    rng = np.random.default_rng(123)
    hq, H, d, p, M = 12, 4, 64, 16, 200
    layers, qs, kps = [], [], []
    for _ in range(3):
        ho, pos, k, v = random_layer(rng, H, rng.integers(180, 320, H), d, dtype=np.float32)
        layers.append((ho, pos, k, v))
        qs.append(rng.standard_normal((hq, p, d)).astype(np.float32))
        kps.append(rng.standard_normal((H, p, d)).astype(np.float32))
    c = _cache_from_layers(gpu, layers, d, torch.float32, slack=32)
    out = gpu.EpisodeCache(c.layers, H, d, c.capacity, torch.float32, "cuda")
    from paper_2509_17396_b200.step import evict_step
    evict_step(c, out, torch.as_tensor(np.stack(qs), device="cuda"), torch.as_tensor(np.stack(kps), device="cuda"),
               [M] * 3, mode="exact_f32", slack=32)
    for l, (ho, pos, k, v) in enumerate(layers):
        s = orc.score_layer_f32(qs[l], k, kps[l], ho, True)
        _, keep = orc.evict_layer(ho, pos, s.astype(np.float64), M)
        ln, opos, ok, ov = out.layer_view(l)
        assert np.array_equal(opos, pos[keep])
        assert np.array_equal(ok.numpy(), k[keep]) and np.array_equal(ov.numpy(), v[keep])
        assert ln.tolist() == [int(keep[ho[h]:ho[h + 1]].sum()) for h in range(H)]


def test_golden_scores_fp64_grids(gpu):
    """score_with_prompt on explicit grids == the reference, bit for bit."""
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_v1.npz"))
    from oracle import oracle as O
    for i in range(int(g["sc_count"])):
        q, k, kp, ho = g[f"sc{i}_q"], g[f"sc{i}_k"], g[f"sc{i}_kp"], g[f"sc{i}_head_off"]
        hq, p, d = q.shape
        H = len(ho) - 1
        G = hq // H
        grids = O.prompt_grids_f64(q, k, kp, ho)
        for agg in (1, 0):
            got = gpu.score_grids(grids, ho, hq, "max" if agg else "avg")
            assert np.array_equal(got, g[f"sc{i}_{agg}_scores"]), (i, agg)

