"""Times the K5 sensitivity reduction at the cfg2 calibration size
(28 layers x 8 kv heads x 32,768 tokens x 128, bf16 K_full and K_block)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_17396_b200 as epk  # noqa: E402

kf = torch.randn(28, 8, 32768, 128, device="cuda").bfloat16()
kb = (kf.float() + 0.3 * torch.randn_like(kf.float())).bfloat16()
for _ in range(2):
    epk.sensitivity_from_keys(kf, kb)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    epk.sensitivity_from_keys(kf, kb)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"sensitivity (cfg2 calibration, 2 x {kf.numel() * 2 / 1e9:.2f} GB bf16): {ms:.3f} ms")
