"""The fused single-kernel block step (csrc/step.cu) against the
multi-launch path and the oracle.

The fused step computes its own scores (bf16 tensor cores, written to
`scores`), selects with the histogram/threshold select and compacts with its
evict warps.  Given those scores, selection + compaction are exact integer
work, so the output cache must equal -- bit for bit -- the generic pooled
select (epk_select_pooled, itself pinned to evict_to_budget by
test_gpu_select.py) + epk_compact run on the same scores.  The scores
themselves are checked against the fp64 oracle (1e-4 relative, bf16 inputs)
and the retained sets against the oracle's (>= 99.9 %).
"""
import numpy as np
import pytest
import torch

from tests.helpers import bf16_round, random_layer

pytestmark = pytest.mark.gpu

SCORE_RTOL = 1e-4
OVERLAP_MIN = 0.999


def _build(gpu, rng, L, Hq, H, p, counts_per_layer, slack, dup_frac=0.0):
    layers, qs, kps = [], [], []
    for l in range(L):
        counts = counts_per_layer[l]
        ho, pos, k, v = random_layer(rng, H, counts, 128, dtype=np.float32)
        k, v = bf16_round(k), bf16_round(v)
        if dup_frac and len(pos) > 4:  # tie stress: identical K rows -> identical scores
            n = len(pos)
            src = rng.choice(n, max(1, int(dup_frac * n)), replace=False)
            dst = rng.choice(n, len(src), replace=False)
            k[dst] = k[src]
        layers.append((ho, pos, k, v))
        qs.append(bf16_round(rng.standard_normal((Hq, p, 128)).astype(np.float32)))
        kps.append(bf16_round(rng.standard_normal((H, p, 128)).astype(np.float32)))
    cap = [int(ho[-1]) + slack * H + 64 for ho, _, _, _ in layers]
    cin = gpu.EpisodeCache(L, H, 128, cap, torch.bfloat16, "cuda")
    cin.load_layers([(np.diff(ho), pos, k, v) for ho, pos, k, v in layers])
    q = torch.as_tensor(np.stack(qs), device="cuda").bfloat16()
    kp = torch.as_tensor(np.stack(kps), device="cuda").bfloat16()
    return layers, qs, kps, cin, q, kp, cap


def _run_fused(gpu, cin, q, kp, budgets, slack, agg, cap, n_max):
    from paper_2509_17396_b200.step import evict_step
    ctx = gpu.default_context(0)
    ctx.set_option(layer_group=0, fused=True)
    cout = gpu.EpisodeCache(cin.layers, cin.kv_heads, 128, cap, torch.bfloat16, "cuda")
    scores = torch.zeros(cin.rows, dtype=torch.float32, device="cuda")
    kept = torch.zeros(cin.layers, dtype=torch.int32, device="cuda")
    evict_step(cin, cout, q, kp, budgets, aggregation=agg, mode="tc_bf16", slack=slack, n_max_per_head=n_max,
               scores=scores, kept_per_layer=kept, ctx=ctx)
    torch.cuda.synchronize()
    ctx.set_option(fused=False)
    ctx.poll_error()
    return cout, scores, kept


def _generic(gpu, cin, scores, budgets, slack, cap):
    keep = gpu.select_pooled(cin, scores, budgets)
    cref = gpu.EpisodeCache(cin.layers, cin.kv_heads, 128, cap, torch.bfloat16, "cuda")
    gpu.compact(cin, keep, cref, slack=slack)
    torch.cuda.synchronize()
    return cref


def _assert_same_cache(a, b):
    assert torch.equal(a.head_off, b.head_off)
    assert torch.equal(a.head_len, b.head_len)
    for l in range(a.layers):
        ra, rb = a.live_rows(l), b.live_rows(l)
        assert torch.equal(a.pos[ra], b.pos[rb]), l
        assert torch.equal(a.k[ra].view(torch.int16), b.k[rb].view(torch.int16)), l
        assert torch.equal(a.v[ra].view(torch.int16), b.v[rb].view(torch.int16)), l


@pytest.mark.parametrize("case", [
    # L, Hq, H, p, counts per layer (ragged, an empty head, a partial tile), M per layer, agg, dup
    (3, 24, 8, 128, [[1280] * 8, [1000, 1500, 0, 77, 1280, 2000, 640, 129], [300] * 8], [1024, 512, 64], "max", 0.0),
    (2, 24, 8, 64, [[900] * 8, [1100, 700, 1300, 500, 900, 900, 1000, 800]], [700, 100000], "max", 0.02),
    (2, 16, 4, 128, [[2500, 1900, 17, 4096], [3000] * 4], [1800, 2500], "avg", 0.0),
    (1, 3, 1, 100, [[5000]], [1234], "max", 0.01),
])
def test_fused_step_bitexact_vs_generic_select_compact(gpu, case):
    L, Hq, H, p, counts, M, agg, dup = case
    rng = np.random.default_rng(sum(M) + p)
    slack = 128
    layers, qs, kps, cin, q, kp, cap = _build(gpu, rng, L, Hq, H, p, counts, slack, dup)
    n_max = max(max(c) for c in counts)
    cout, scores, kept = _run_fused(gpu, cin, q, kp, M, slack, agg, cap, n_max)
    cref = _generic(gpu, cin, scores, M, slack, cap)
    _assert_same_cache(cout, cref)
    exp_kept = [min(int(sum(c)), H * m) for c, m in zip(counts, M)]
    assert kept.cpu().tolist() == exp_kept


def test_fused_step_scores_and_overlap_vs_oracle(gpu, orc):
    rng = np.random.default_rng(11)
    L, Hq, H, p, M, slack = 2, 24, 8, 128, 1024, 256
    counts = [[1280] * H, [1100, 1400, 1280, 1200, 1350, 1280, 1300, 1330]]
    layers, qs, kps, cin, q, kp, cap = _build(gpu, rng, L, Hq, H, p, counts, slack)
    cout, scores, _ = _run_fused(gpu, cin, q, kp, [M] * L, slack, "max", cap, 1400)
    sc = scores.cpu().numpy()
    for l, (ho, pos, k, v) in enumerate(layers):
        exp = orc.score_layer_f64(qs[l].astype(np.float64), k.astype(np.float64), kps[l].astype(np.float64), ho, True)
        b = int(cin.layer_base[l])
        got = sc[b:b + len(pos)]
        assert (np.abs(got - exp) / exp).max() < SCORE_RTOL
        _, keep = orc.evict_layer(ho, pos, exp, M)
        ref = [pos[ho[h]:ho[h + 1]][keep[ho[h]:ho[h + 1]]].tolist() for h in range(H)]
        got_pos = cout.retained_positions()[l]
        inter = sum(len(set(a) & set(r)) for a, r in zip(got_pos, ref))
        assert sum(len(a) for a in got_pos) == H * M
        assert inter / (H * M) >= OVERLAP_MIN


def test_fused_step_chained_episode_matches_layer_group_path(gpu):
    """Chained block steps (append -> fused step) keep the cache consistent:
    every step's output equals generic select+compact on its own scores."""
    from paper_2509_17396_b200.step import evict_step
    rng = np.random.default_rng(5)
    L, Hq, H, p, M, B = 2, 24, 8, 128, 512, 256
    cap = H * (M + B)
    ctx = gpu.default_context(0)
    ctx.set_option(layer_group=0, fused=True)
    a = gpu.EpisodeCache(L, H, 128, cap, torch.bfloat16, "cuda")
    b = gpu.EpisodeCache(L, H, 128, cap, torch.bfloat16, "cuda")
    a.set_regions(M + B)
    start = 0
    for step in range(5):
        kn = torch.as_tensor(bf16_round(rng.standard_normal((L, H, B, 128)).astype(np.float32)), device="cuda").bfloat16()
        vn = torch.as_tensor(bf16_round(rng.standard_normal((L, H, B, 128)).astype(np.float32)), device="cuda").bfloat16()
        q = torch.as_tensor(bf16_round(rng.standard_normal((L, Hq, p, 128)).astype(np.float32)), device="cuda").bfloat16()
        kp = torch.as_tensor(bf16_round(rng.standard_normal((L, H, p, 128)).astype(np.float32)), device="cuda").bfloat16()
        posn = torch.arange(start, start + B, dtype=torch.int32, device="cuda")
        start += B
        gpu.append_to_cache(a, kn, vn, posn, ctx=ctx)
        torch.cuda.synchronize()
        ctx.poll_error()
        scores = torch.zeros(a.rows, dtype=torch.float32, device="cuda")
        evict_step(a, b, q, kp, [M] * L, mode="tc_bf16", slack=B, n_max_per_head=M + B, scores=scores, ctx=ctx)
        torch.cuda.synchronize()
        ctx.poll_error()
        cref = _generic(gpu, a, scores, [M] * L, B, [cap] * L)
        ctx.poll_error()
        _assert_same_cache(b, cref)
        assert b.entries_per_layer() == [min(H * M, (step + 1) * H * B)] * L
        a, b = b, a
    ctx.set_option(fused=False)
