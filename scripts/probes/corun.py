"""Probe: can the compaction gather of one layer group co-run with the scorer
(P1 + P2) of the next on the same SMs?  Times, at the cfg2 shape:
  score alone (P1 + P2 over L layers), compaction alone (count/plan/gather of
  an independent cache), and both launched together on two streams.
Usage: python scripts/probes/corun.py [variant.so] [layers]"""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2509_17396_b200 as epk  # noqa: E402
from paper_2509_17396_b200 import _lib  # noqa: E402
from paper_2509_17396_b200.context import Context  # noqa: E402

if len(sys.argv) > 1 and sys.argv[1].endswith(".so"):
    _lib.LIB_PATH = os.path.abspath(sys.argv[1])
L = int(sys.argv[2]) if len(sys.argv) > 2 else 28
H, Hq, d, p, n_h, M = 8, 24, 128, 128, 10240, 8192
dev = torch.device("cuda", 0)


def cache():
    c = epk.EpisodeCache(L, H, d, [H * n_h] * L, torch.bfloat16, dev)
    c.k.normal_()
    c.v.normal_()
    c.pos.copy_(torch.arange(n_h, device=dev, dtype=torch.int32).repeat(L * H))
    c.head_off.copy_((torch.arange(H + 1, device=dev, dtype=torch.int32) * n_h).repeat(L, 1))
    c.head_len.fill_(n_h)
    return c


A, C = cache(), cache()
D = epk.EpisodeCache(L, H, d, [H * (M + 2048)] * L, torch.bfloat16, dev)
q = torch.randn(L, Hq, p, d, device=dev).bfloat16()
kp = torch.randn(L, H, p, d, device=dev).bfloat16()
s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
c1, c2 = Context(0, s1), Context(0, s2)
scores = torch.empty(A.rows, device=dev)
with torch.cuda.stream(s2):
    sc = epk.score_with_prompt(C, q, kp, ctx=c2)
    keep = epk.select_pooled(C, sc, [M] * L, ctx=c2)
torch.cuda.synchronize()


def score():
    epk.score_with_prompt(A, q, kp, out=scores, n_max_per_head=n_h, ctx=c1)


def comp():
    epk.compact(C, keep, D, slack=2048, ctx=c2)


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e3


def both():
    ev = torch.cuda.Event()
    ev.record(torch.cuda.current_stream())
    s1.wait_event(ev)
    s2.wait_event(ev)
    score()
    comp()
    e1, e2 = torch.cuda.Event(), torch.cuda.Event()
    e1.record(s1)
    e2.record(s2)
    torch.cuda.current_stream().wait_event(e1)
    torch.cuda.current_stream().wait_event(e2)


def score_sync():
    score()


def comp_sync():
    comp()


def both_rev():
    ev = torch.cuda.Event()
    ev.record(torch.cuda.current_stream())
    s1.wait_event(ev)
    s2.wait_event(ev)
    comp()
    score()
    e1, e2 = torch.cuda.Event(), torch.cuda.Event()
    e1.record(s1)
    e2.record(s2)
    torch.cuda.current_stream().wait_event(e1)
    torch.cuda.current_stream().wait_event(e2)


def timeline(first_comp):
    """start / end of each stream's work relative to a common start (ms)."""
    ev = torch.cuda.Event(enable_timing=True)
    ev.record(torch.cuda.current_stream())
    s1.wait_event(ev)
    s2.wait_event(ev)
    a0, a1, b0, b1 = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    if first_comp:
        b0.record(s2); comp(); b1.record(s2)
        a0.record(s1); score(); a1.record(s1)
    else:
        a0.record(s1); score(); a1.record(s1)
        b0.record(s2); comp(); b1.record(s2)
    torch.cuda.synchronize()
    return (ev.elapsed_time(a0), ev.elapsed_time(a1), ev.elapsed_time(b0), ev.elapsed_time(b1))


ts = timed(score_sync)
tc = timed(comp_sync)
tb = timed(both)
tr = timed(both_rev)
tl1 = timeline(False)
tl2 = timeline(True)
c1.profile(True)
score()
rec = c1.profile_records()
c1.profile(False)
print(f"lib {os.path.basename(_lib.LIB_PATH)} L={L}: score {ts:.3f} ms ({', '.join(f'{n} {m:.3f}' for n, m in rec)}), "
      f"compaction {tc:.3f} ms, sum {ts + tc:.3f}, co-run {tb:.3f} ms (compaction first {tr:.3f})\n"
      f"   timeline score-first: score {tl1[0]:.3f}-{tl1[1]:.3f} comp {tl1[2]:.3f}-{tl1[3]:.3f}; "
      f"comp-first: score {tl2[0]:.3f}-{tl2[1]:.3f} comp {tl2[2]:.3f}-{tl2[3]:.3f}")
