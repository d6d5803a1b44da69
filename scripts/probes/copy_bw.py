"""HBM copy ceiling on this B200: cudaMemcpy D2D and torch copy_ of 0.95 GB
(= one cfg2 gather's K or V bytes), read+write bytes counted."""
import torch

n = 948_011_008  # bytes: half of the cfg2 gather's 1.896 GB algorithmic traffic
a = torch.empty(n, dtype=torch.uint8, device="cuda")
b = torch.empty(n, dtype=torch.uint8, device="cuda")
a.fill_(1)
for _ in range(3):
    b.copy_(a)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 20
e0.record()
for _ in range(reps):
    b.copy_(a)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
print(f"D2D copy {n/1e9:.2f} GB: {ms:.3f} ms -> {2*n/ms/1e6:.0f} GB/s (read+write)")
