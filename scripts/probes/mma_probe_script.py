"""Diagnostic (not a test): tcgen05 MMA issue ceiling on this B200."""
import sys
sys.path.insert(0, '.')
import paper_2509_17396_b200 as epk
from paper_2509_17396_b200 import _lib
ctx = epk.default_context(0)
iters = 4000
for n in (64, 128, 192, 256):
    for drain in (0, 1):
        ctx.profile(True)
        for _ in range(4):
            _lib.call("epk_debug_mma_rate", ctx.handle, n, iters, drain)
        recs = ctx.profile_records(); ctx.profile(False)
        ms = sorted(r[1] for r in recs)[1]
        flops = 2.0 * 128 * n * 128 * iters * 148
        print(f"N={n} drain={drain}: {ms:.3f} ms  {flops / ms / 1e9:.0f} TFLOP/s  "
              f"{ms * 1e-3 * 1.965e9 / iters:.0f} cycles/job (at 1965 MHz)")


# two-SM pairs (cta_group::2, M = 256): flops per SM comparable with the lines above
for n in (128, 256):
    ctx.profile(True)
    for _ in range(4):
        _lib.call("epk_debug_mma2sm_rate", ctx.handle, n, iters)
    recs = ctx.profile_records(); ctx.profile(False)
    ms = sorted(r[1] for r in recs)[1]
    flops = 2.0 * 256 * n * 128 * iters * 74
    print(f"2SM M=256 N={n}: {ms:.3f} ms  {flops / ms / 1e9:.0f} TFLOP/s  "
          f"{ms * 1e-3 * 1.965e9 / iters:.0f} cycles/job (pair, at 1965 MHz)")
