"""Edge cases of the C ABI that must fail closed or keep
evict_to_budget's semantics at the extremes:

* a layer budget of 0 keeps nothing (kvcache.hpp:180-190 with no pins) on the
  default tensor-core step (threshold select) as on the generic select;
* an output cache too small for the kept rows raises EPK_ERR_ARG and the
  gather writes nothing past the offending layer (the next layer's rows stay
  intact and correct), on the generic compaction and on the default step
  (whose threshold select plans the compaction);
* the exact-f32 scorer refuses a head longer than n_max_per_head instead of
  overrunning its scratch;
* epk_append honours its slack argument;
* two contexts on two host threads (the per-(thread, GPU) contract of epk.h)
  score concurrently and give the sequential bits.
"""
import threading

import numpy as np
import pytest
import torch

from tests.helpers import bf16_round

pytestmark = pytest.mark.gpu


def _cache(gpu, rng, counts_per_layer, slack, dtype=torch.bfloat16, d=128, cap_extra=0):
    per = []
    H = len(counts_per_layer[0])
    for c in counts_per_layer:
        c = np.asarray(c, np.int64)
        n = int(c.sum())
        pos = np.concatenate([np.sort(rng.choice(4 * max(1, int(c.max())) + 8, int(x), replace=False))
                              for x in c]).astype(np.int64)
        per.append((c, pos, bf16_round(rng.standard_normal((n, d)).astype(np.float32)),
                    bf16_round(rng.standard_normal((n, d)).astype(np.float32))))
    cap = [int(c.sum()) + slack * H + cap_extra for c, _, _, _ in per]
    cin = gpu.EpisodeCache(len(per), H, d, cap, dtype, "cuda")
    cin.load_layers(per, slack=slack)
    return cin, cap


def test_zero_budget_keeps_nothing(gpu, orc):
    from paper_2509_17396_b200.step import evict_step
    rng = np.random.default_rng(0)
    L, H, Hq, p, slack = 3, 4, 8, 16, 8
    counts = [[90, 70, 0, 40], [60, 60, 60, 60], [5, 0, 0, 1]]
    budgets = [0, 20, 0]
    cin, cap = _cache(gpu, rng, counts, slack)
    q = torch.randn(L, Hq, p, 128, device="cuda").bfloat16()
    kp = torch.randn(L, H, p, 128, device="cuda").bfloat16()
    # poison the threshold state a previous layer would leave behind
    out = gpu.EpisodeCache(L, H, 128, cap, torch.bfloat16, "cuda")
    scores = torch.zeros(cin.rows, dtype=torch.float32, device="cuda")
    kept = torch.full((L,), -1, dtype=torch.int32, device="cuda")
    for _ in range(2):  # second run reuses the step buffers of the first
        evict_step(cin, out, q, kp, budgets, mode="tc_bf16", slack=slack, scores=scores, kept_per_layer=kept)
        torch.cuda.synchronize()
        gpu.default_context(0).poll_error()
        assert kept.cpu().tolist() == [0, 80, 0]
        assert out.head_len[0].sum().item() == 0 and out.head_len[2].sum().item() == 0
    ref = gpu.EpisodeCache(L, H, 128, cap, torch.bfloat16, "cuda")
    keep = gpu.select_pooled(cin, scores, budgets)
    gpu.compact(cin, keep, ref, slack=slack)
    torch.cuda.synchronize()
    assert out.retained_positions() == ref.retained_positions()
    # the generic select agrees with the reference semantics (oracle) at budget 0
    for l in (0, 2):
        ln, pos, _, _ = cin.layer_view(l)
        ho = np.concatenate([[0], np.cumsum(ln)]).astype(np.int64)
        st, k_or = orc.evict_layer(ho, pos.astype(np.int64), np.ones(len(pos)), 0)
        assert st == 0 and k_or.sum() == 0
        assert keep[int(cin.layer_base[l]):int(cin.layer_base[l + 1])].sum().item() == 0


def test_compact_overflow_fails_closed(gpu):
    rng = np.random.default_rng(1)
    H, slack = 2, 4
    counts = [[50, 50], [30, 30]]
    cin, cap = _cache(gpu, rng, counts, slack)
    keep = torch.zeros(cin.rows, dtype=torch.uint8, device="cuda")
    for l in range(2):
        keep[cin.live_rows(l)] = 1  # keep everything
    small = [60, 30 * 2 + slack * H]  # layer 0 cannot hold 100 rows; layer 1 fits exactly
    out = gpu.EpisodeCache(2, H, 128, small, torch.bfloat16, "cuda")
    out.k.fill_(7.0)
    gpu.compact(cin, keep, out, slack=slack)
    torch.cuda.synchronize()
    with pytest.raises(gpu.Error):
        gpu.default_context(0).poll_error()
    # layer 0 is left empty and nothing landed past its 60 rows
    assert out.head_len[0].sum().item() == 0
    assert bool((out.k[int(out.layer_base[1]):][out.pos[int(out.layer_base[1]):] < 0] == 7.0).all())
    # layer 1 is intact and correct
    assert out.retained_positions()[1] == cin.retained_positions()[1]
    ra, rb = out.live_rows(1), cin.live_rows(1)
    assert torch.equal(out.k[ra].view(torch.int16), cin.k[rb].view(torch.int16))


def test_tc_step_overflow_fails_closed(gpu):
    """The default tensor-core step plans the compaction inside its threshold
    select: an output layer too small for its kept rows is flagged
    (EPK_ERR_ARG), left empty and never written past, and the other layers
    equal the generic select + compaction on the step's own scores."""
    from paper_2509_17396_b200.step import evict_step
    rng = np.random.default_rng(11)
    L, H, Hq, p, slack = 3, 4, 8, 16, 8
    counts = [[300, 250, 0, 90], [120, 120, 120, 120], [40, 41, 42, 43]]
    budgets = [100, 60, 50]  # layer 2 is under budget: everything kept
    cin, cap = _cache(gpu, rng, counts, slack)
    small = list(cap)
    small[1] = 60 * H + slack * H - 1  # one row short of layer 1's kept rows + slack
    q = torch.randn(L, Hq, p, 128, device="cuda").bfloat16()
    kp = torch.randn(L, H, p, 128, device="cuda").bfloat16()
    out = gpu.EpisodeCache(L, H, 128, small, torch.bfloat16, "cuda")
    out.k.fill_(7.0)
    scores = torch.zeros(cin.rows, dtype=torch.float32, device="cuda")
    evict_step(cin, out, q, kp, budgets, mode="tc_bf16", slack=slack, scores=scores)
    torch.cuda.synchronize()
    with pytest.raises(gpu.Error):
        gpu.default_context(0).poll_error()
    assert out.head_len[1].sum().item() == 0
    b1, b2 = int(out.layer_base[1]), int(out.layer_base[2])
    assert bool((out.k[b1:b2] == 7.0).all())  # nothing landed in (or past) layer 1
    ref = gpu.EpisodeCache(L, H, 128, cap, torch.bfloat16, "cuda")
    gpu.compact(cin, gpu.select_pooled(cin, scores, budgets), ref, slack=slack)
    torch.cuda.synchronize()
    for l in (0, 2):
        assert out.retained_positions()[l] == ref.retained_positions()[l]
        ra, rb = out.live_rows(l), ref.live_rows(l)
        assert torch.equal(out.k[ra].view(torch.int16), ref.k[rb].view(torch.int16))
        assert torch.equal(out.v[ra].view(torch.int16), ref.v[rb].view(torch.int16))


def test_f32_scorer_refuses_short_n_max(gpu):
    rng = np.random.default_rng(2)
    cin, _ = _cache(gpu, rng, [[40, 300]], 0, dtype=torch.float32)
    q = torch.randn(1, 4, 8, 128, device="cuda")
    kp = torch.randn(1, 2, 8, 128, device="cuda")
    sc = gpu.score_with_prompt(cin, q, kp, "max", mode="exact_f32", n_max_per_head=300)
    torch.cuda.synchronize()
    gpu.default_context(0).poll_error()
    out = torch.full((cin.rows,), -5.0, device="cuda")
    gpu.score_with_prompt(cin, q, kp, "max", mode="exact_f32", n_max_per_head=100, out=out)
    torch.cuda.synchronize()
    with pytest.raises(gpu.Error):
        gpu.default_context(0).poll_error()
    # the short head is scored as before, the long one untouched
    assert torch.equal(out[:40], sc[:40])
    assert bool((out[40:340] == -5.0).all())


def test_append_slack_checked(gpu):
    H, L, d = 2, 1, 128
    c = gpu.EpisodeCache(L, H, d, [2 * 16], torch.bfloat16, "cuda")
    c.set_regions(16)
    k = torch.randn(L, H, 10, d, device="cuda").bfloat16()
    pos = torch.arange(10, device="cuda", dtype=torch.int32)
    with pytest.raises(gpu.Error):
        gpu.append_to_cache(c, k, k, pos, slack=8)  # block of 10 > declared slack 8
    gpu.append_to_cache(c, k, k, pos, slack=16)
    torch.cuda.synchronize()
    assert c.head_len.cpu().tolist() == [[10, 10]]
    gpu.append_to_cache(c, k, k, pos + 10)  # 20 > the 16-row region: refused on the device
    torch.cuda.synchronize()
    with pytest.raises(gpu.Error):
        gpu.default_context(0).poll_error()
    assert c.head_len.cpu().tolist() == [[10, 10]]


def test_two_contexts_two_threads(gpu):
    from paper_2509_17396_b200.context import Context
    rng = np.random.default_rng(3)
    cin, _ = _cache(gpu, rng, [[700, 500, 650, 0]] * 3, 0)
    q = torch.randn(3, 12, 64, 128, device="cuda").bfloat16()
    kp = torch.randn(3, 4, 64, 128, device="cuda").bfloat16()
    ref = gpu.score_with_prompt(cin, q, kp, "max", mode="tc_bf16").clone()
    torch.cuda.synchronize()
    outs = [None, None]

    def work(i):
        torch.cuda.set_device(0)
        s = torch.cuda.Stream()
        ctx = Context(0, s)
        with torch.cuda.stream(s):
            o = torch.zeros(cin.rows, device="cuda")
            for _ in range(5):
                gpu.score_with_prompt(cin, q, kp, "max", mode="tc_bf16", out=o, ctx=ctx)
            s.synchronize()
        outs[i] = o
        ctx.close()

    th = [threading.Thread(target=work, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    live = torch.cat([cin.live_rows(l) for l in range(3)])
    for o in outs:
        assert torch.equal(o[live].view(torch.int32), ref[live].view(torch.int32))


def test_nan_scores_are_refused(gpu):
    """SURVEY 7 hard part 5: a NaN score has no place in evict_to_budget's
    order (kvcache.hpp:181-185); the scorers and the generic select flag it
    (deferred EPK_ERR_NAN) instead of selecting on garbage."""
    from paper_2509_17396_b200.step import evict_step
    rng = np.random.default_rng(6)
    cin, cap = _cache(gpu, rng, [[100, 80]], 4)
    cin.k[3, 0] = float("nan")
    q = torch.randn(1, 4, 8, 128, device="cuda").bfloat16()
    kp = torch.randn(1, 2, 8, 128, device="cuda").bfloat16()
    out = gpu.EpisodeCache(1, 2, 128, cap, torch.bfloat16, "cuda")
    evict_step(cin, out, q, kp, [50], mode="tc_bf16", slack=4)
    torch.cuda.synchronize()
    with pytest.raises(gpu.Error, match="NaN"):
        gpu.default_context(0).poll_error()
    scores = torch.rand(cin.rows, device="cuda")
    scores[int(cin.live_rows(0)[7])] = float("nan")
    with pytest.raises(gpu.Error, match="NaN"):
        gpu.select_pooled(cin, scores, [50])
