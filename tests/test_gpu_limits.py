"""The default tensor-core block step (epk_evict_step: P1 -> P2 with fused
histograms -> threshold select + compaction plan -> gather) at the edges of its
layout limits -- 128 layers (kMaxLayers), 64 kv heads (kMaxHeads), heads that
are empty or under budget, a whole layer under budget -- bit-exact against the
generic pooled select + compaction (themselves pinned to evict_to_budget by
test_gpu_select.py) on the scores the step itself produced."""
import numpy as np
import pytest
import torch

from tests.helpers import bf16_round

pytestmark = pytest.mark.gpu


def _cache(gpu, rng, L, H, counts, slack):
    per = []
    for l in range(L):
        c = np.asarray(counts[l], np.int64)
        n = int(c.sum())
        pos = np.concatenate([np.sort(rng.choice(4 * max(1, int(c.max())) + 8, int(x), replace=False))
                              for x in c]).astype(np.int64) if n else np.zeros(0, np.int64)
        per.append((c, pos, bf16_round(rng.standard_normal((n, 128)).astype(np.float32)),
                    bf16_round(rng.standard_normal((n, 128)).astype(np.float32))))
    cap = [int(c.sum()) + slack * H for c, _, _, _ in per]
    cin = gpu.EpisodeCache(L, H, 128, cap, torch.bfloat16, "cuda")
    cin.load_layers(per, slack=slack)
    return cin, cap


def _check_step(gpu, cin, cap, Hq, p, budgets, slack, rng):
    from paper_2509_17396_b200.step import evict_step
    L, H = cin.layers, cin.kv_heads
    q = torch.as_tensor(bf16_round(rng.standard_normal((L, Hq, p, 128)).astype(np.float32)), device="cuda").bfloat16()
    kp = torch.as_tensor(bf16_round(rng.standard_normal((L, H, p, 128)).astype(np.float32)), device="cuda").bfloat16()
    out = gpu.EpisodeCache(L, H, 128, cap, torch.bfloat16, "cuda")
    scores = torch.zeros(cin.rows, dtype=torch.float32, device="cuda")
    kept = torch.zeros(L, dtype=torch.int32, device="cuda")
    evict_step(cin, out, q, kp, budgets, mode="tc_bf16", slack=slack, scores=scores, kept_per_layer=kept)
    torch.cuda.synchronize()
    ref = gpu.EpisodeCache(L, H, 128, cap, torch.bfloat16, "cuda")
    gpu.compact(cin, gpu.select_pooled(cin, scores, budgets), ref, slack=slack)
    torch.cuda.synchronize()
    assert torch.equal(out.head_off, ref.head_off) and torch.equal(out.head_len, ref.head_len)
    for l in range(L):
        ra, rb = out.live_rows(l), ref.live_rows(l)
        assert torch.equal(out.pos[ra], ref.pos[rb]), l
        assert torch.equal(out.k[ra].view(torch.int16), ref.k[rb].view(torch.int16)), l
        assert torch.equal(out.v[ra].view(torch.int16), ref.v[rb].view(torch.int16)), l
    live = cin.head_len.sum(dim=1).cpu().numpy()
    assert kept.cpu().tolist() == [int(min(n, H * b)) for n, b in zip(live, budgets)]


def test_step_128_layers(gpu):
    rng = np.random.default_rng(128)
    L, H = 128, 2
    counts = [[int(rng.integers(0, 400)), int(rng.integers(0, 400))] for _ in range(L)]
    budgets = [int(rng.integers(1, 300)) for _ in range(L)]
    cin, cap = _cache(gpu, rng, L, H, counts, slack=16)
    _check_step(gpu, cin, cap, 6, 32, budgets, 16, rng)


def test_step_64_heads(gpu):
    rng = np.random.default_rng(64)
    L, H = 2, 64
    counts = [[int(x) for x in rng.integers(0, 300, H)], [150] * H]
    counts[0][5] = 0
    budgets = [100, 200]  # layer 1 is under budget: everything kept
    cin, cap = _cache(gpu, rng, L, H, counts, slack=8)
    _check_step(gpu, cin, cap, 64, 16, budgets, 8, rng)


def test_tc_step_with_pins_equals_generic(gpu):
    """Pins take the tc step off the fused threshold select (epk_evict_step's
    generic branch: tc scores -> pooled select with pins -> compaction); the
    result must equal select_pooled + compact with the same pins on the
    step's own scores."""
    from paper_2509_17396_b200.step import evict_step
    rng = np.random.default_rng(77)
    L, H, slack = 2, 4, 8
    counts = [[300, 250, 0, 90], [120, 120, 120, 120]]
    cin, cap = _cache(gpu, rng, L, H, counts, slack)
    pins = {0, 1, 5}
    budgets = [100, 60]
    q = torch.as_tensor(bf16_round(rng.standard_normal((L, 8, 16, 128)).astype(np.float32)), device="cuda").bfloat16()
    kp = torch.as_tensor(bf16_round(rng.standard_normal((L, H, 16, 128)).astype(np.float32)), device="cuda").bfloat16()
    out = gpu.EpisodeCache(L, H, 128, cap, torch.bfloat16, "cuda")
    scores = torch.zeros(cin.rows, dtype=torch.float32, device="cuda")
    evict_step(cin, out, q, kp, budgets, pinned=pins, mode="tc_bf16", slack=slack, scores=scores)
    torch.cuda.synchronize()
    ref = gpu.EpisodeCache(L, H, 128, cap, torch.bfloat16, "cuda")
    gpu.compact(cin, gpu.select_pooled(cin, scores, budgets, pins), ref, slack=slack)
    torch.cuda.synchronize()
    assert out.retained_positions() == ref.retained_positions()
    for l in range(L):
        present = {p for h in range(H) for p in cin.retained_positions()[l][h]}
        kept = {p for h in range(H) for p in out.retained_positions()[l][h]}
        assert (pins & present) <= kept
