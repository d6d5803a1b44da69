"""TMA gather probe (epk_debug_tma_gather): the cfg2 compaction's K/V traffic
moved by tile::gather4 loads + bulk stores on a subset of SMs.  Checks the
result against torch indexing, then times 148 / 64 / 32 / 16 SMs."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2509_17396_b200 as epk  # noqa: E402
from paper_2509_17396_b200 import _lib  # noqa: E402

rows = 28 * 8 * 10240
k = torch.randn(rows, 128, device="cuda").bfloat16()
v = torch.randn(rows, 128, device="cuda").bfloat16()
g = torch.Generator(device="cuda").manual_seed(0)
keep = (torch.rand(rows, device="cuda", generator=g) < 0.8).to(torch.uint8)
cnt = keep.view(-1, 128).sum(dim=1, dtype=torch.int32)
prefix = (torch.cumsum(cnt, 0, dtype=torch.int32) - cnt).contiguous()
kept = int(cnt.sum())
kout = torch.empty(kept, 128, device="cuda", dtype=torch.bfloat16)
vout = torch.empty_like(kout)
ctx = epk.default_context(0)


def run(sms):
    _lib.call("epk_debug_tma_gather", ctx.handle, C.c_void_p(k.data_ptr()), C.c_void_p(v.data_ptr()), rows,
              C.c_void_p(keep.data_ptr()), C.c_void_p(prefix.data_ptr()), C.c_void_p(kout.data_ptr()),
              C.c_void_p(vout.data_ptr()), sms)


run(148)
torch.cuda.synchronize()
idx = keep.nonzero().squeeze(1)
assert torch.equal(kout.view(torch.int16), k[idx].view(torch.int16)) and torch.equal(vout.view(torch.int16), v[idx].view(torch.int16))
print("tma gather correct")
moved = kept * 256 * 2 * 2  # K and V, read + write
for sms in (148, 96, 64, 32, 16):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    run(sms)
    e0.record()
    for _ in range(5):
        run(sms)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"tma gather on {sms:3d} SMs: {ms:.3f} ms, {moved / ms / 1e6:.0f} GB/s (kept-row bytes read+written)")
