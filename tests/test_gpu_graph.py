"""CUDA-graph capture of the chained block loop: eight
block steps of append_to_cache (epk_append) + the default tensor-core step
(epk_evict_step) ping-ponging between two caches, captured once and
replayed, give the eager run's bits; cfg1 (1 layer, 16K context, block 512,
M = 2,048, p = 64) replays its 32-block episode with no host launches."""
import time

import pytest
import torch

pytestmark = pytest.mark.gpu


def _setup(gpu, L, H, Hq, d, p, M, B, nblk, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    cap = [H * (M + B)] * L
    bufs = [gpu.EpisodeCache(L, H, d, cap, torch.bfloat16, "cuda") for _ in range(2)]
    for c in bufs:
        c.set_regions(M + B)
    ks = [torch.randn(L, H, B, d, device="cuda", generator=g).bfloat16() for _ in range(nblk)]
    vs = [torch.randn(L, H, B, d, device="cuda", generator=g).bfloat16() for _ in range(nblk)]
    poss = [torch.arange(b * B, (b + 1) * B, device="cuda", dtype=torch.int32) for b in range(nblk)]
    q = torch.randn(L, Hq, p, d, device="cuda", generator=g).bfloat16()
    kp = torch.randn(L, H, p, d, device="cuda", generator=g).bfloat16()
    return bufs, ks, vs, poss, q, kp


def _episode(gpu, bufs, ks, vs, poss, q, kp, M, B, plans, ctx):
    from paper_2509_17396_b200.step import evict_step
    L = bufs[0].layers
    for b in range(len(ks)):
        cur = b % 2
        gpu.append_to_cache(bufs[cur], ks[b], vs[b], poss[b], slack=B, ctx=ctx)
        evict_step(bufs[cur], bufs[1 - cur], q, kp, [M] * L, mode="tc_bf16", slack=B, n_max_per_head=M + B,
                   plan=plans[cur], ctx=ctx)


def _reset(bufs, M, B):
    for c in bufs:
        c.set_regions(M + B)


def test_graph_replay_equals_eager(gpu):
    from paper_2509_17396_b200.step import StepPlan
    L, H, Hq, d, p, M, B, nblk = 2, 8, 24, 128, 64, 256, 128, 8
    bufs, ks, vs, poss, q, kp = _setup(gpu, L, H, Hq, d, p, M, B, nblk, 1)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        ctx = gpu.default_context(0)
        plans = [StepPlan(bufs[0], bufs[1], [M] * L), StepPlan(bufs[1], bufs[0], [M] * L)]
        _episode(gpu, bufs, ks, vs, poss, q, kp, M, B, plans, ctx)  # eager (also sizes every workspace)
        s.synchronize()
        ctx.poll_error()
        eager = bufs[nblk % 2]
        ref_pos = eager.retained_positions()
        ref_k = [eager.k[eager.live_rows(l)].clone() for l in range(L)]
        _reset(bufs, M, B)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            _episode(gpu, bufs, ks, vs, poss, q, kp, M, B, plans, ctx)
        for _ in range(2):  # replays are repeatable
            _reset(bufs, M, B)
            graph.replay()
            s.synchronize()
            ctx.poll_error()
            got = bufs[nblk % 2]
            assert got.retained_positions() == ref_pos
            for l in range(L):
                assert torch.equal(got.k[got.live_rows(l)].view(torch.int16), ref_k[l].view(torch.int16))


def test_cfg1_episode_graph_timing(gpu):
    """cfg1's 32-block episode: eager vs graph replay (printed; the graph
    must not be slower)."""
    from paper_2509_17396_b200.step import StepPlan
    L, H, Hq, d, p, M, B, nblk = 1, 8, 24, 128, 64, 2048, 512, 32
    bufs, ks, vs, poss, q, kp = _setup(gpu, L, H, Hq, d, p, M, B, nblk, 2)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        ctx = gpu.default_context(0)
        plans = [StepPlan(bufs[0], bufs[1], [M] * L), StepPlan(bufs[1], bufs[0], [M] * L)]
        _episode(gpu, bufs, ks, vs, poss, q, kp, M, B, plans, ctx)
        s.synchronize()
        ref = bufs[nblk % 2].retained_positions()
        graph = torch.cuda.CUDAGraph()
        _reset(bufs, M, B)
        with torch.cuda.graph(graph, stream=s):
            _episode(gpu, bufs, ks, vs, poss, q, kp, M, B, plans, ctx)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        times = {}
        for mode in ("eager", "graph", "eager", "graph"):
            _reset(bufs, M, B)
            s.synchronize()
            e0.record(s)
            if mode == "graph":
                graph.replay()
            else:
                _episode(gpu, bufs, ks, vs, poss, q, kp, M, B, plans, ctx)
            e1.record(s)
            s.synchronize()
            times[mode] = e0.elapsed_time(e1)
        assert bufs[nblk % 2].retained_positions() == ref
    print(f"cfg1 32-block episode: eager {times['eager']:.3f} ms, graph replay {times['graph']:.3f} ms "
          f"({times['eager'] / nblk * 1e3:.1f} / {times['graph'] / nblk * 1e3:.1f} us per block)")
    assert times["graph"] <= times["eager"] * 1.1
