"""Times the fp32 parity path (K1' exact scorer + generic pooled select +
compaction) for one cfg2 block step: 28 layers x 8 heads x 10,240 live rows."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_17396_b200 as epk  # noqa: E402
from paper_2509_17396_b200.step import evict_step  # noqa: E402

L, H, Hq, d, n, M, p, B = 28, 8, 24, 128, 10240, 8192, 128, 2048
a = epk.EpisodeCache(L, H, d, [H * (n + B)] * L, torch.float32, "cuda")
b = epk.EpisodeCache(L, H, d, [H * (n + B)] * L, torch.float32, "cuda")
a.set_regions(n + B)
a.head_len.fill_(n)
a.k.normal_()
a.v.normal_()
a.pos.copy_((torch.arange(a.rows, device="cuda") % (n + B)).to(torch.int32))
q = torch.randn(L, Hq, p, d, device="cuda")
kp = torch.randn(L, H, p, d, device="cuda")
for _ in range(2):
    evict_step(a, b, q, kp, [M] * L, mode="exact_f32", slack=B, n_max_per_head=n)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 5
e0.record()
for _ in range(reps):
    evict_step(a, b, q, kp, [M] * L, mode="exact_f32", slack=B, n_max_per_head=n)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
print(f"fp32 parity step (cfg2 shape): {ms:.2f} ms/step = {L * H * n / ms * 1e3:.3g} units/s")
