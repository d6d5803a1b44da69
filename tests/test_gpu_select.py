"""K2 (pooled / per-head selection) + K3 (compaction) against the oracle's
evict_to_budget restatement -- bit-exact, through the C ABI.  Mirrors
test_kvcache.cpp (direct top-k, 200-trial global-sort oracle, determinism,
pin overflow, under budget) and acceptance C3 (500 trials)."""
import numpy as np
import pytest
import torch

from tests.helpers import composite_topk, quantised_scores, random_layer

pytestmark = pytest.mark.gpu


def _device_layer(epk, ho, pos, k, v, dtype=torch.float64, slack_cap=0):
    H = len(ho) - 1
    n = int(ho[-1])
    d = k.shape[1]
    c = epk.EpisodeCache(1, H, d, [max(n, 1) + slack_cap], dtype, "cuda")
    c.load_layers([(np.diff(ho), pos, k, v)])
    return c


def _evict_gpu(epk, ho, pos, scores, budget, pins=(), k=None, v=None, dtype=torch.float64, score_dtype=torch.float64):
    n = len(pos)
    if k is None:
        k = np.zeros((n, 2))
        v = np.zeros((n, 2))
    c = _device_layer(epk, ho, pos, k, v, dtype)
    sc = torch.as_tensor(np.asarray(scores), device="cuda").to(score_dtype)
    keep = epk.select_pooled(c, sc, [budget], set(pins), synchronous=True)
    out = epk.EpisodeCache(1, c.kv_heads, c.head_dim, c.capacity, dtype, "cuda")
    epk.compact(c, keep, out, 0)
    torch.cuda.synchronize()
    return keep.cpu().numpy().astype(bool), out


def test_direct_topk(gpu):
    keep, out = _evict_gpu(gpu, np.array([0, 4]), np.arange(4), [5., 1., 9., 2.], 2)
    assert np.nonzero(keep)[0].tolist() == [0, 2]
    assert out.retained_positions() == [[[0, 2]]]


def test_200_trials_global_sort(gpu, orc):
    rng = np.random.default_rng(5)
    for trial in range(200):
        H = 1 + trial % 2
        budget = int(1 + rng.integers(0, 4))
        ho, pos, _, _ = random_layer(rng, H, [6] * H, 1, pos_space=6)
        sc = quantised_scores(rng, len(pos))
        pins = {0} if (trial % 3 == 0 and H * budget > H) else set()
        keep, _ = _evict_gpu(gpu, ho, pos, sc, budget, pins)
        st, ok = orc.evict_layer(ho, pos, sc, budget, pins)
        assert np.array_equal(keep, ok), trial
        assert np.array_equal(keep, composite_topk(ho, pos, sc, budget, pins))


def test_500_trials_c3(gpu, orc):
    rng = np.random.default_rng(2024)
    for trial in range(500):
        H = int(1 + rng.integers(0, 4))
        budget = int(1 + rng.integers(0, 6))
        block = int(1 + rng.integers(0, 8))
        n = int(1 + rng.integers(0, budget + block))
        ho = np.arange(H + 1) * n
        pos = np.tile(np.arange(n), H)
        sc = rng.integers(0, 5, H * n).astype(np.float64)
        pins = {0} if trial % 4 == 0 else set()
        keep, _ = _evict_gpu(gpu, ho, pos, sc, budget, pins)
        st, ok = orc.evict_layer(ho, pos, sc, budget, pins)
        assert np.array_equal(keep, ok), trial


def test_golden_evictions(gpu):
    import os
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_v1.npz"))
    for i in range(int(g["ev_count"])):
        if int(g[f"ev{i}_status"]) != 0 or len(g[f"ev{i}_pos"]) == 0:
            continue
        keep, _ = _evict_gpu(gpu, g[f"ev{i}_head_off"], g[f"ev{i}_pos"], g[f"ev{i}_scores"], int(g[f"ev{i}_budget"]),
                             set(g[f"ev{i}_pins"].tolist()))
        assert np.array_equal(keep, g[f"ev{i}_keep"]), i


@pytest.mark.parametrize("score_dtype", [torch.float32, torch.float64])
def test_random_real_scores_and_compaction_bitwise(gpu, orc, score_dtype):
    rng = np.random.default_rng(11)
    for trial in range(30):
        H = int(rng.integers(1, 9))
        counts = rng.integers(0, 300, H)
        ho, pos, k, v = random_layer(rng, H, counts, 16)
        sc = rng.random(len(pos)).astype(np.float32).astype(np.float64)
        if trial % 5 == 0:
            sc = np.round(sc * 4) / 4  # ties
        budget = int(rng.integers(1, 200))
        keep, out = _evict_gpu(gpu, ho, pos, sc, budget, (), k, v, torch.float64, score_dtype)
        st, ok = orc.evict_layer(ho, pos, sc, budget)
        assert np.array_equal(keep, ok)
        ln, opos, ok_k, ok_v = out.layer_view(0)
        assert np.array_equal(opos, pos[ok]) and np.array_equal(ok_k.numpy(), k[ok]) and np.array_equal(ok_v.numpy(), v[ok])
        # per-head counts of the compacted CSR
        exp_counts = [int(ok[ho[h]:ho[h + 1]].sum()) for h in range(H)]
        assert ln.tolist() == exp_counts


def test_negative_zero_and_negative_scores(gpu, orc):
    # -0.0 == +0.0 in the reference comparator: the tie falls to the position
    ho = np.array([0, 3, 6])
    pos = np.array([0, 1, 2, 0, 1, 2])
    sc = np.array([-0.0, 0.0, -1.5, 0.0, -0.0, -2.0])
    for budget in (1, 2):
        keep, _ = _evict_gpu(gpu, ho, pos, sc, budget)
        _, ok = orc.evict_layer(ho, pos, sc, budget)
        assert np.array_equal(keep, ok)


def test_all_tied_deterministic(gpu, orc):
    ho = np.array([0, 6, 12])
    pos = np.tile(np.arange(6), 2)
    sc = np.ones(12)
    a, _ = _evict_gpu(gpu, ho, pos, sc, 2)
    b, _ = _evict_gpu(gpu, ho, pos, sc, 2)
    _, ok = orc.evict_layer(ho, pos, sc, 2)
    assert np.array_equal(a, b) and np.array_equal(a, ok)


def test_pin_overflow_raises(gpu):
    with pytest.raises(gpu.Error, match="exceed layer budget"):
        _evict_gpu(gpu, np.array([0, 3]), np.arange(3), np.zeros(3), 1, {0, 1, 2})


def test_under_budget_unchanged(gpu):
    keep, out = _evict_gpu(gpu, np.array([0, 3]), np.arange(3), [0., 1., 2.], 4)
    assert keep.all() and out.retained_positions() == [[[0, 1, 2]]]


def test_multilayer_ragged_with_slack(gpu, orc):
    """Several layers with different budgets; output regions leave slack."""
    rng = np.random.default_rng(21)
    L, H, d = 5, 4, 32
    layers = []
    for l in range(L):
        counts = rng.integers(50, 200, H)
        layers.append(random_layer(rng, H, counts, d))
    budgets = [int(b) for b in rng.integers(10, 80, L)]
    cap = [int(ho[-1]) + 64 * H for ho, _, _, _ in layers]
    c = gpu.EpisodeCache(L, H, d, cap, torch.float32, "cuda")
    c.load_layers([(np.diff(ho), pos, k, v) for ho, pos, k, v in layers])
    sc_all = torch.zeros(c.rows, dtype=torch.float32, device="cuda")
    exp = []
    for l, (ho, pos, k, v) in enumerate(layers):
        sc = rng.random(len(pos)).astype(np.float32)
        b = int(c.layer_base[l])
        sc_all[b:b + len(pos)] = torch.as_tensor(sc, device="cuda")
        exp.append(orc.evict_layer(ho, pos, sc.astype(np.float64), budgets[l])[1])
    keep = gpu.select_pooled(c, sc_all, budgets)
    out = gpu.EpisodeCache(L, H, d, cap, torch.float32, "cuda")
    gpu.compact(c, keep, out, slack=64)
    for l, (ho, pos, k, v) in enumerate(layers):
        ln, opos, ok_k, _ = out.layer_view(l)
        assert np.array_equal(opos, pos[exp[l]])
        assert np.array_equal(ok_k.numpy(), k[exp[l]].astype(np.float32))
        off = out.head_off[l].cpu().numpy()
        assert np.all(np.diff(off) - ln == 64)  # slack after every head


def test_per_head_topk_vs_reference_semantics(gpu, orc):
    rng = np.random.default_rng(3)
    for trial in range(40):
        ho, pos, _, _ = random_layer(rng, 3, rng.integers(0, 40, 3), 1)
        sc = quantised_scores(rng, len(pos), 3)
        kk = int(rng.integers(0, 30))
        c = _device_layer(gpu, ho, pos, np.zeros((len(pos), 2)), np.zeros((len(pos), 2)))
        keep = gpu.select_per_head(c, torch.as_tensor(sc, device="cuda"), [kk]).cpu().numpy().astype(bool)
        assert np.array_equal(keep[:len(pos)], orc.topk_per_head(ho, sc, kk))


def test_dropin_layercache_api(gpu, orc):
    """The reference-signature drop-in: LayerCache + per-head score maps."""
    rng = np.random.default_rng(7)
    H, budget = 2, 3
    cache = gpu.LayerCache.empty(H, budget)
    scores = [dict(), dict()]
    for h in range(H):
        for p in range(8):
            cache.heads[h].append(gpu.KVEntry(p, rng.standard_normal(4).tolist(), rng.standard_normal(4).tolist()))
            scores[h][p] = float(rng.uniform())
    out = gpu.evict_to_budget(cache, scores)
    assert out.entry_count() == 6
    for head in out.heads:
        assert all(head[i - 1].position < head[i].position for i in range(1, len(head)))
    ho = np.array([0, 8, 16])
    pos = np.tile(np.arange(8), 2)
    sc = np.array([scores[h][p] for h in range(2) for p in range(8)])
    _, ok = orc.evict_layer(ho, pos, sc, budget)
    got = [e.position for e in out.heads[0]], [e.position for e in out.heads[1]]
    assert got[0] == pos[:8][ok[:8]].tolist() and got[1] == pos[8:][ok[8:]].tolist()
    with pytest.raises(gpu.DimensionError):
        gpu.evict_to_budget(cache, [scores[0]])
    bad = [dict(scores[0]), dict(scores[1])]
    del bad[1][3]
    with pytest.raises(gpu.DimensionError, match="missing score"):
        gpu.evict_to_budget(cache, bad)


def test_full_size_layer_properties(gpu):
    """cfg2 layer shape (81,920 live entries, keep 65,536): exact count,
    composite-key threshold property checked with torch sort."""
    H, n_h, M = 8, 10240, 8192
    torch.manual_seed(0)
    c = gpu.EpisodeCache(1, H, 128, [H * (M + 2048)], torch.bfloat16, "cuda")
    ho = np.arange(H + 1) * n_h
    pos = np.tile(np.arange(n_h), H)
    c.load_layers([(np.full(H, n_h), pos, np.zeros((H * n_h, 128), np.float32), np.zeros((H * n_h, 128), np.float32))])
    sc = torch.rand(c.rows, device="cuda", dtype=torch.float32)
    sc[: H * n_h: 7] = 0.5  # ties
    keep = gpu.select_pooled(c, sc, [M]).bool()[: H * n_h]
    assert int(keep.sum()) == H * M
    s = sc[: H * n_h].double()
    head = torch.arange(H, device="cuda").repeat_interleave(n_h)
    p = torch.as_tensor(pos, device="cuda")
    # composite order: score desc, pos asc, head asc
    key = torch.stack([-s, p.double(), head.double()], 1).cpu().numpy()
    order = np.lexsort((key[:, 2], key[:, 1], key[:, 0]))
    exp = np.zeros(H * n_h, bool)
    exp[order[: H * M]] = True
    assert np.array_equal(keep.cpu().numpy(), exp)
