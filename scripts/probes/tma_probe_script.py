import torch, ctypes as C, sys
sys.path.insert(0, '.')
import paper_2509_17396_b200 as epk
from paper_2509_17396_b200 import _lib
ctx = epk.default_context(0)
rows = 28*8*10240*2
k = torch.randn(rows, 128, device='cuda').bfloat16()
for box in (64, 128, 256):
    for st in (2, 3, 4, 6, 8, 12):
        if st*box*256 > 200*1024: continue
        for grid in (148, 296):
            if grid == 296 and st*box*256*2 > 220*1024: continue
            ctx.profile(True)
            for _ in range(5):
                _lib.call("epk_debug_tma_stream", ctx.handle, C.c_void_p(k.data_ptr()), rows, box, st, grid)
            recs = ctx.profile_records(); ctx.profile(False)
            ms = sorted(r[1] for r in recs)[2]
            print(f"box={box:3d} stages={st:2d} grid={grid} inflight/SM={st*box*256*(grid//148)//1024}KB  {rows*256/ms/1e6:8.0f} GB/s")
