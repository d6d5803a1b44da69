"""K4 per-kernel device time of one epk_kmeans call (2,048 x 1,024, k = 4 / 8)
from the context's live CUDA-event profile, next to the call's wall time and
the points' H2D copy (the Python wrapper uploads the host array)."""
import collections
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_17396_b200 as epk  # noqa: E402

rng = np.random.default_rng(0)
ctx = epk.default_context(0)
out = {}
for dim in (1024, 256):
    centers = rng.standard_normal((8, dim))
    pts = centers[rng.integers(0, 8, 2048)] + 0.8 * rng.standard_normal((2048, dim))
    for k in (4, 8):
        epk.kmeans(pts, k, seed=1, ctx=ctx)
        torch.cuda.synchronize()
        ctx.profile(True)
        t = time.perf_counter()
        r = epk.kmeans(pts, k, seed=1, ctx=ctx)
        wall = (time.perf_counter() - t) * 1e3
        recs = ctx.profile_records()
        ctx.profile(False)
        agg = collections.defaultdict(lambda: [0, 0.0])
        for name, ms in recs:
            agg[name][0] += 1
            agg[name][1] += ms
        t = time.perf_counter()
        for _ in range(5):
            d = torch.as_tensor(pts, device="cuda")
        torch.cuda.synchronize()
        h2d = (time.perf_counter() - t) / 5 * 1e3
        out[f"kmeans_2048x{dim}_k{k}"] = {
            "iterations": r.iterations, "wall_ms_profiled": round(wall, 3), "points_h2d_ms": round(h2d, 3),
            "kernels": {n: {"launches": c, "ms": round(v, 4)} for n, (c, v) in agg.items()},
            "device_ms_total": round(sum(v for _, v in agg.values()), 4)}
print(json.dumps(out, indent=1))
