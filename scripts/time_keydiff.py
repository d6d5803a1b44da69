"""Times the KeyDiff scorer (K6) + pooled select + compaction at the cfg2 shape."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_17396_b200 as epk  # noqa: E402

L, H, d, n, M = 28, 8, 128, 10240, 8192
c = epk.EpisodeCache(L, H, d, [H * n] * L, torch.bfloat16, "cuda")
c.set_regions(n)
c.k.copy_(torch.randn(c.rows, d, device="cuda").bfloat16())
c.head_len.fill_(n)
c.pos.copy_(torch.arange(c.rows, device="cuda", dtype=torch.int32) % n)
out = epk.EpisodeCache(L, H, d, [H * n] * L, torch.bfloat16, "cuda")
sc = torch.zeros(c.rows, dtype=torch.float64, device="cuda")
for _ in range(3):
    epk.keydiff_scores(c, out=sc)
torch.cuda.synchronize()
e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
reps = 10
e0.record()
for _ in range(reps):
    epk.keydiff_scores(c, out=sc)
e1.record()
for _ in range(reps):
    keep = epk.select_pooled(c, sc, [M] * L)
    epk.compact(c, keep, out, slack=0)
e2.record()
torch.cuda.synchronize()
ks = e0.elapsed_time(e1) / reps
ss = e1.elapsed_time(e2) / reps
print(f"keydiff scores: {ks:.3f} ms/step ({c.rows * d * 2 / ks / 1e6:.0f} GB/s of K), "
      f"select+compact (fp64 generic path): {ss:.3f} ms/step")
