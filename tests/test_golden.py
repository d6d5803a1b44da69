"""The oracle against golden fixtures generated from the reference itself
(tests/golden/make_golden.py).  Runs anywhere (no /root/reference needed)."""
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_v1.npz")


@pytest.fixture(scope="module")
def g():
    return np.load(GOLDEN)


def test_evict_fixtures(orc, g):
    for i in range(int(g["ev_count"])):
        st, keep = orc.evict_layer(g[f"ev{i}_head_off"], g[f"ev{i}_pos"], g[f"ev{i}_scores"], int(g[f"ev{i}_budget"]),
                                   set(g[f"ev{i}_pins"].tolist()))
        if int(g[f"ev{i}_status"]) == -2:
            assert st == -2
        else:
            assert np.array_equal(keep, g[f"ev{i}_keep"]), i


def test_score_fixtures_bitwise(orc, g):
    for i in range(int(g["sc_count"])):
        for agg in (1, 0):
            s = orc.score_layer_f64(g[f"sc{i}_q"], g[f"sc{i}_k"], g[f"sc{i}_kp"], g[f"sc{i}_head_off"], bool(agg))
            assert np.array_equal(s, g[f"sc{i}_{agg}_scores"]), (i, agg)


def test_kmeans_fixtures_bitwise(orc, g):
    for i in range(int(g["km_count"])):
        a, c, it, sse = orc.kmeans(g[f"km{i}_pts"], int(g[f"km{i}_k"]), int(g[f"km{i}_seed"]))
        assert np.array_equal(a, g[f"km{i}_assign"]) and np.array_equal(c, g[f"km{i}_cent"])
        assert it == int(g[f"km{i}_iters"]) and np.array_equal(sse, g[f"km{i}_sse"])


def test_allocate_fixtures(orc, g):
    for i in range(int(g["al_count"])):
        b, w = orc.allocate(g[f"al{i}_s"], int(g[f"al{i}_M"]), float(g[f"al{i}_alpha"]))
        assert np.array_equal(b, g[f"al{i}_b"]) and np.array_equal(w, g[f"al{i}_w"])


def test_sensitivity_fixture(orc, g):
    sigma, skipped = orc.sensitivity(g["sens_kf"], g["sens_kb"])
    assert np.array_equal(sigma, g["sens_sigma"]) and skipped == int(g["sens_skipped"])


def test_keydiff_fixtures_bitwise(orc, g):
    for i in range(int(g["kd_count"])):
        s = orc.keydiff_layer(g[f"kd{i}_k"], g[f"kd{i}_head_off"])
        assert np.array_equal(s, g[f"kd{i}_scores"]), i


def test_trace_fixture(g):
    assert g["bp_c2_series"].tolist() == [3, 1, 4, 1, 4, 1]
    assert g["bp_alloc_counts"].tolist() == [4, 12]


def test_expf_contract(orc):
    """EPK-F32 v1 exp: <= 1 ulp from the correctly rounded value on the
    softmax domain, exact 1 at 0, 0 below -103.97."""
    x = np.linspace(-87.0, 0.0, 400001).astype(np.float32)
    y = orc.expf(x)
    cr = np.exp(x.astype(np.float64)).astype(np.float32)
    assert np.max(np.abs(y.view(np.int32).astype(np.int64) - cr.view(np.int32))) <= 1
    assert orc.expf(np.array([0.0], np.float32))[0] == 1.0
    assert orc.expf(np.array([-104.0], np.float32))[0] == 0.0


def test_threaded_scorers_equal_single_threaded(orc, g):
    """The multi-threaded restatements (used by the benchmark-scale GPU parity
    tests) give the single-threaded bits: golden fp64 fixtures, ragged heads,
    p not a multiple of 4, both aggregations, fp64 and EPK-F32."""
    for i in range(int(g["sc_count"])):
        for agg in (1, 0):
            s = orc.score_layer_f64_mt(g[f"sc{i}_q"], g[f"sc{i}_k"], g[f"sc{i}_kp"], g[f"sc{i}_head_off"], bool(agg),
                                       threads=3)
            assert np.array_equal(s, g[f"sc{i}_{agg}_scores"]), (i, agg)
    rng = np.random.default_rng(5)
    for hq, hkv, p, counts in ((6, 2, 7, [33, 0]), (8, 4, 5, [10, 70, 1, 64]), (3, 3, 1, [5, 6, 7])):
        ho = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        q = rng.standard_normal((hq, p, 16))
        k = rng.standard_normal((int(ho[-1]), 16))
        kp = rng.standard_normal((hkv, p, 16))
        for agg in (True, False):
            assert np.array_equal(orc.score_layer_f64_mt(q, k, kp, ho, agg, threads=4),
                                  orc.score_layer_f64(q, k, kp, ho, agg))
            q32, k32, kp32 = q.astype(np.float32), k.astype(np.float32), kp.astype(np.float32)
            assert np.array_equal(orc.score_layer_f32_mt(q32, k32, kp32, ho, agg, threads=2).view(np.uint32),
                                  orc.score_layer_f32(q32, k32, kp32, ho, agg).view(np.uint32))


def test_maxpool_restatement_vs_loop(orc):
    """oracle.maxpool_scores (the opt-in smoothing's checker) against a plain
    per-element loop: windows clipped at head boundaries, empty heads."""
    rng = np.random.default_rng(2)
    ho = np.array([0, 7, 7, 20, 21])
    s = rng.random(21).astype(np.float32)
    for k in (1, 3, 5, 9, 41):
        got = orc.maxpool_scores(ho, s, k)
        for h in range(4):
            for j in range(ho[h], ho[h + 1]):
                lo, hi = max(ho[h], j - k // 2), min(ho[h + 1] - 1, j + k // 2)
                assert got[j] == s[lo:hi + 1].max()
