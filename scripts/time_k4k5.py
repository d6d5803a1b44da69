"""K4 / K5 timing: k-means over 2,048 segment embeddings of dim
1,024 (Qwen3-Embedding-0.6B) and 256 (the reference HashEmbedder),
k = 4 and 8 -- end to end (host seeding + Lloyd on the device) and per Lloyd
iteration; and the layer-sensitivity reduction at the cfg2 calibration size
(28 x 8 x 32,768 x 128 bf16 key pairs), with its per-kernel split."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_17396_b200 as epk  # noqa: E402

out = {}
rng = np.random.default_rng(0)
for dim in (1024, 256):
    centers = rng.standard_normal((8, dim))
    pts = centers[rng.integers(0, 8, 2048)] + 0.8 * rng.standard_normal((2048, dim))
    for k in (4, 8):
        epk.kmeans(pts, k, seed=1)
        torch.cuda.synchronize()
        reps = 5
        t = time.perf_counter()
        for _ in range(reps):
            r = epk.kmeans(pts, k, seed=1)
        ms = (time.perf_counter() - t) / reps * 1e3
        out[f"kmeans_2048x{dim}_k{k}"] = {"ms_end_to_end": ms, "iterations": r.iterations,
                                          "us_per_lloyd_iteration": 1e3 * ms / max(1, r.iterations)}
kf = torch.randn(28, 8, 32768, 128, device="cuda").bfloat16()
kb = (kf.float() + 0.3 * torch.randn_like(kf.float())).bfloat16()
ctx = epk.default_context(0)
for _ in range(2):
    epk.sensitivity_from_keys(kf, kb)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    epk.sensitivity_from_keys(kf, kb)
e1.record()
torch.cuda.synchronize()
ctx.profile(True)
epk.sensitivity_from_keys(kf, kb)
rec = ctx.profile_records()
ctx.profile(False)
gb = 2 * kf.numel() * 2 / 1e9
ms = e0.elapsed_time(e1) / 5
out["sensitivity_cfg2_calibration"] = {"ms": ms, "bytes_gb": gb, "achieved_gbs": gb / ms * 1e3,
                                       "kernels_ms": {n: m for n, m in rec}}
print(json.dumps(out, indent=1))
