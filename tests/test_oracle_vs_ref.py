"""Pins the CPU oracle (oracle/epk_oracle.cpp) to the reference headers
themselves (oracle/_ref/libepkref.so, compiled from /root/reference).

Mirrors the reference's own module tests: test_kvcache.cpp (global-sort
oracle, 200 trials; direct top-k; pin overflow), acceptance_test.cpp C3
(500 trials) and C2 (3,1,4,1,4,1), test_scoring.cpp, test_clustering.cpp,
test_allocation.cpp.
"""
import numpy as np
import pytest

from tests.helpers import composite_topk, quantised_scores, random_layer


@pytest.mark.parametrize("agg", [True, False])
@pytest.mark.parametrize("shape", [(6, 2, 16, 5, [13, 9]), (3, 1, 8, 1, [7]), (8, 4, 32, 7, [0, 5, 11, 2]),
                                   (24, 8, 128, 4, [40] * 8)])
def test_score_f64_bitwise(ref, agg, shape):
    hq, H, d, p, counts = shape
    rng = np.random.default_rng(hash((hq, H, d, p)) % 2**32)
    ho, pos, k, _ = random_layer(rng, H, counts, d)
    q = rng.standard_normal((hq, p, d))
    kp = rng.standard_normal((H, p, d))
    a = ref.score_layer_f64(q, k, kp, ho, agg)
    b = ref.ref_score_layer_f64(q, k, kp, ho, pos, agg)
    assert np.array_equal(a, b)


def test_score_f32_close_to_f64(ref):
    rng = np.random.default_rng(5)
    ho, pos, k, _ = random_layer(rng, 8, [300] * 8, 128)
    q = rng.standard_normal((24, 64, 128))
    kp = rng.standard_normal((8, 64, 128))
    ref64 = ref.ref_score_layer_f64(q, k, kp, ho, pos, True)
    f32 = ref.score_layer_f32(q.astype(np.float32), k.astype(np.float32), kp.astype(np.float32), ho, True)
    assert np.max(np.abs(f32 - ref64) / ref64) < 1e-5


def test_score_grids_hand_grid(ref):
    # test_scoring.cpp:71-95 hand grid, plus "head 1 wins" (:136-149)
    grid = np.array([[0.10, 0.20, 0.05, 0.40], [0.30, 0.10, 0.20, 0.15], [0.05, 0.50, 0.10, 0.05]])
    full = np.concatenate([grid, np.zeros((3, 3))], axis=1)
    ho = np.array([0, 4])
    pos = np.arange(4)
    mx = ref.ref_score_grids([full], ho, pos, 1, True)
    av = ref.ref_score_grids([full], ho, pos, 1, False)
    assert np.allclose(mx, grid.max(0), atol=1e-15)
    assert np.allclose(av, grid.sum(0) / 3, atol=1e-15)
    g = [np.array([[0.1 * (j + 1) + 0.5 * qh for j in range(3)] + [0, 0]] * 2) for qh in range(2)]
    s = ref.ref_score_grids(g, np.array([0, 3]), np.arange(3), 2, True)
    assert np.array_equal(s, np.array([0.1 * (j + 1) + 0.5 for j in range(3)]))


def test_evict_direct_topk(ref):
    # test_kvcache.cpp:85-96: scores (5,1,9,2), M=2 -> {0,2}
    st, keep = ref.evict_layer(np.array([0, 4]), np.arange(4), np.array([5., 1., 9., 2.]), 2)
    assert st == 0 and np.nonzero(keep)[0].tolist() == [0, 2]
    keep2, _, _ = ref.ref_evict_layer(np.array([0, 4]), np.arange(4), np.array([5., 1., 9., 2.]), 2)
    assert np.array_equal(keep, keep2)


def test_evict_200_trials_global_sort(ref):
    # test_kvcache.cpp:117-142 analogue (quantised scores, pins)
    rng = np.random.default_rng(5)
    for trial in range(200):
        H = 1 + trial % 2
        budget = 1 + rng.integers(0, 4)
        ho, pos, _, _ = random_layer(rng, H, [6] * H, 1, pos_space=6)
        sc = quantised_scores(rng, len(pos))
        pins = {0} if (trial % 3 == 0 and H * budget > H) else set()
        st, keep = ref.evict_layer(ho, pos, sc, budget, pins)
        rk, _, _ = ref.ref_evict_layer(ho, pos, sc, budget, pins)
        assert np.array_equal(keep, rk)
        assert np.array_equal(keep, composite_topk(ho, pos, sc, budget, pins))


def test_evict_500_trials_c3(ref):
    # acceptance_test.cpp:174-239 analogue: heads 1..4, budget 1..6, block 1..8
    rng = np.random.default_rng(2024)
    for trial in range(500):
        H = 1 + rng.integers(0, 4)
        budget = 1 + rng.integers(0, 6)
        block = 1 + rng.integers(0, 8)
        n = 1 + rng.integers(0, budget + block)
        ho = np.arange(H + 1) * n
        pos = np.tile(np.arange(n), H)
        sc = rng.integers(0, 5, H * n).astype(np.float64)
        pins = {0} if trial % 4 == 0 else set()
        st, keep = ref.evict_layer(ho, pos, sc, budget, pins)
        rk, _, _ = ref.ref_evict_layer(ho, pos, sc, budget, pins)
        assert np.array_equal(keep, rk), trial


def test_evict_pin_overflow_and_under_budget(ref):
    ho, pos = np.array([0, 3]), np.arange(3)
    st, _ = ref.evict_layer(ho, pos, np.zeros(3), 1, {0, 1, 2})
    assert st == -2
    with pytest.raises(ref.RefError) as ei:
        ref.ref_evict_layer(ho, pos, np.zeros(3), 1, {0, 1, 2})
    assert "exceed layer budget" in ei.value.msg
    st, keep = ref.evict_layer(ho, pos, np.zeros(3), 4)
    assert st == 1 and keep.all()


def test_evict_keeps_kv_rows_bitwise(ref):
    rng = np.random.default_rng(9)
    ho, pos, k, v = random_layer(rng, 3, [10, 7, 12], 16)
    sc = rng.random(len(pos))
    keep, counts, (ko, vo, po) = ref.ref_evict_layer(ho, pos, sc, 5, k=k, v=v)
    assert np.array_equal(ko, k[keep]) and np.array_equal(vo, v[keep]) and np.array_equal(po, pos[keep])


def test_topk_per_head_vs_ref(ref):
    rng = np.random.default_rng(3)
    for trial in range(50):
        ho, pos, _, _ = random_layer(rng, 2, [9, 5], 1)
        sc = quantised_scores(rng, len(pos), 3)
        kk = int(rng.integers(0, 8))
        keep = ref.topk_per_head(ho, sc, kk)
        for h in range(2):
            idx = ref.ref_top_k_indices(sc[ho[h]:ho[h + 1]], kk)
            assert np.nonzero(keep[ho[h]:ho[h + 1]])[0].tolist() == idx.tolist()


@pytest.mark.parametrize("n,dim,k,seed", [(200, 8, 4, 7), (64, 3, 1, 1), (12, 2, 12, 5), (500, 32, 8, 11)])
def test_kmeans_bitwise(ref, n, dim, k, seed):
    rng = np.random.default_rng(seed)
    pts = rng.standard_normal((n, dim))
    a = ref.kmeans(pts, k, seed)
    b = ref.ref_kmeans(pts, k, seed)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and a[2] == b[2]
    assert np.array_equal(a[3], b[3])


def test_kmeans_duplicate_points_repair(ref):
    pts = np.repeat(np.random.default_rng(0).standard_normal((3, 4)), 5, axis=0)
    pts = np.concatenate([pts, pts[:1]])
    a = ref.kmeans(pts, 6, 3)
    b = ref.ref_kmeans(pts, 6, 3)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_sensitivity_and_allocate(ref):
    sig, sk, kf, kb = ref.ref_measure_sensitivity(3, 4, 2, 8, 3, 64, 5, 16, 4)
    s2, sk2 = ref.sensitivity(kf, kb)
    assert np.array_equal(sig, s2) and sk == sk2
    rng = np.random.default_rng(1)
    for _ in range(100):
        L = int(rng.integers(1, 30))
        s = rng.random(L) * (rng.random(L) > 0.2)
        M = int(rng.integers(1, 300))
        alpha = float(rng.choice([0.0, 0.5, 1.0, 1.1, 2.0]))
        try:
            b1, w1 = ref.allocate(s, M, alpha)
        except ValueError:
            with pytest.raises(ref.RefError):
                ref.ref_allocate(s, M, alpha)
            continue
        b2, w2 = ref.ref_allocate(s, M, alpha)
        assert np.array_equal(b1, b2) and np.array_equal(w1, w2)
    b, _ = ref.ref_allocate(np.array([0.1, 0.3]), 100, 1.0)  # test_allocation.cpp:128-133
    assert b.tolist() == [50, 150]


def test_block_prefill_trace_c2(ref):
    # acceptance C2 / test_blockprefill.cpp:70-79
    series, ev, nb, counts, _ = ref.ref_block_prefill(1, 1, 1, 8, 3, 9, 2, 1, 3, [7, 21, 42])
    assert series.tolist() == [3, 1, 4, 1, 4, 1] and nb == 3


def test_keydiff_bitwise(ref):
    """KeyDiff restatement (scoring.hpp:186-221) vs the reference: ragged heads,
    empty head, zero key, zero-anchor head, bf16-valued keys."""
    import torch
    rng = np.random.default_rng(7)
    for trial in range(12):
        H = int(rng.integers(1, 9))
        counts = rng.integers(0, 300, H)
        d = int(rng.choice([4, 64, 128]))
        ho, pos, k, _ = random_layer(rng, H, counts, d)
        if trial % 3 == 1:
            k = torch.as_tensor(k, dtype=torch.float32).bfloat16().double().numpy()
        if trial % 4 == 2 and len(pos):
            k[rng.integers(0, len(pos))] = 0.0
        if trial % 5 == 3 and counts[0] > 0:
            k[ho[0]:ho[1]] = 0.0
        assert np.array_equal(ref.keydiff_layer(k, ho), ref.ref_keydiff_layer(k, ho, pos)), trial
