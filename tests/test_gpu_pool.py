"""Opt-in 1-D max-pool smoothing (north_star's "max-pool smoothing"; the
reference has none): epk_pool_scores bit-exact vs the numpy
restatement oracle.maxpool_scores (itself checked against a plain loop in
tests/test_golden.py), and the block step with EPK_OPT_POOL_KERNEL equal to
pool -> pooled select -> compaction on the step's own scores; kernel 1 is the
reference's semantics."""
import numpy as np
import pytest
import torch

from tests.helpers import bf16_round

pytestmark = pytest.mark.gpu


def _cache(gpu, rng, counts, slack):
    per = []
    H = len(counts[0])
    for c in counts:
        c = np.asarray(c, np.int64)
        n = int(c.sum())
        pos = np.concatenate([np.sort(rng.choice(4 * max(1, int(c.max())) + 8, int(x), replace=False))
                              for x in c]).astype(np.int64)
        per.append((c, pos, bf16_round(rng.standard_normal((n, 128)).astype(np.float32)),
                    bf16_round(rng.standard_normal((n, 128)).astype(np.float32))))
    cap = [int(c.sum()) + slack * H for c, _, _, _ in per]
    cin = gpu.EpisodeCache(len(per), H, 128, cap, torch.bfloat16, "cuda")
    cin.load_layers(per, slack=slack)
    return cin, cap


@pytest.mark.parametrize("kernel", [1, 3, 7, 31])
def test_pool_scores_bitwise(gpu, orc, kernel):
    rng = np.random.default_rng(kernel)
    cin, _ = _cache(gpu, rng, [[300, 0, 5, 1000], [64, 64, 64, 64]], slack=9)
    scores = torch.rand(cin.rows, device="cuda")
    pooled = gpu.pool_scores(cin, scores, kernel)
    torch.cuda.synchronize()
    for l in range(cin.layers):
        rows = cin.live_rows(l)
        ln = cin.head_len[l].cpu().numpy()
        ho = np.concatenate([[0], np.cumsum(ln)])
        exp = orc.maxpool_scores(ho, scores[rows].cpu().numpy(), kernel)
        assert np.array_equal(pooled[rows].cpu().numpy().view(np.uint32), exp.view(np.uint32))
    with pytest.raises(gpu.Error):
        gpu.pool_scores(cin, scores, 4)


@pytest.mark.parametrize("kernel", [1, 7])
def test_step_with_pooling_equals_pool_then_select(gpu, kernel):
    from paper_2509_17396_b200.step import evict_step
    rng = np.random.default_rng(10 + kernel)
    L, H, Hq, p, slack, M = 3, 4, 12, 32, 16, 150
    cin, cap = _cache(gpu, rng, [[400, 200, 333, 0], [180] * 4, [90, 500, 10, 250]], slack)
    q = torch.randn(L, Hq, p, 128, device="cuda").bfloat16()
    kp = torch.randn(L, H, p, 128, device="cuda").bfloat16()
    ctx = gpu.default_context(0)
    ctx.set_option(pool_kernel=kernel)
    try:
        out = gpu.EpisodeCache(L, H, 128, cap, torch.bfloat16, "cuda")
        scores = torch.zeros(cin.rows, device="cuda")
        evict_step(cin, out, q, kp, [M] * L, mode="tc_bf16", slack=slack, scores=scores, ctx=ctx)
        torch.cuda.synchronize()
        ctx.poll_error()
    finally:
        ctx.set_option(pool_kernel=1)
    pooled = gpu.pool_scores(cin, scores, kernel) if kernel > 1 else scores
    ref = gpu.EpisodeCache(L, H, 128, cap, torch.bfloat16, "cuda")
    gpu.compact(cin, gpu.select_pooled(cin, pooled, [M] * L), ref, slack=slack)
    torch.cuda.synchronize()
    assert out.retained_positions() == ref.retained_positions()
    assert torch.equal(out.head_len, ref.head_len)
