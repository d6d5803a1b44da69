"""Diagnostic (not a test): tcgen05 MMA issue ceiling on this B200."""
import sys
sys.path.insert(0, '.')
import paper_2509_17396_b200 as epk
from paper_2509_17396_b200 import _lib
ctx = epk.default_context(0)
iters = 4000
for n in (128, 256):
    for drain in (0, 1):
        ctx.profile(True)
        for _ in range(4):
            _lib.call("epk_debug_mma_rate", ctx.handle, n, iters, drain)
        recs = ctx.profile_records(); ctx.profile(False)
        ms = sorted(r[1] for r in recs)[1]
        flops = 2.0 * 128 * n * 128 * iters * 148
        print(f"N={n} drain={drain}: {ms:.3f} ms  {flops / ms / 1e9:.0f} TFLOP/s  "
              f"{ms * 1e-3 * 1.965e9 / iters:.0f} cycles/job (at 1965 MHz)")

import torch
rows = 28 * 8 * 10240
k = torch.randn(rows, 128, device='cuda').bfloat16()
import ctypes as C
for nq in (1, 3):
    for st in (2, 3):
        for drain in (0, 1):
            if nq * 32768 + st * 65536 > 226 * 1024:
                continue
            ctx.profile(True)
            for _ in range(4):
                _lib.call("epk_debug_mma_stream", ctx.handle, C.c_void_p(k.data_ptr()), rows, nq, st, drain)
            recs = ctx.profile_records(); ctx.profile(False)
            ms = sorted(r[1] for r in recs)[1]
            flops = 2.0 * 128 * rows * 128 * nq
            print(f"stream nq={nq} stages={st} drain={drain}: {ms:.3f} ms  K {rows * 256 / ms / 1e6:.0f} GB/s  "
                  f"{flops / ms / 1e9:.0f} TFLOP/s")
