import sys; sys.path.insert(0, '.')
import numpy as np, torch
import paper_2509_17396_b200 as gpu
from paper_2509_17396_b200.step import evict_step
from tests.helpers import bf16_round
rng = np.random.default_rng(5)
L, Hq, H, p, M, B = 2, 24, 8, 128, 512, 256
cap = H * (M + B)
ctx = gpu.default_context(0)
ctx.set_option(layer_group=0)
a = gpu.EpisodeCache(L, H, 128, cap, torch.bfloat16, "cuda")
b = gpu.EpisodeCache(L, H, 128, cap, torch.bfloat16, "cuda")
a.set_regions(M + B)
start = 0
for step in range(5):
    kn = torch.randn(L, H, B, 128, device="cuda").bfloat16(); vn = torch.randn_like(kn)
    q = torch.randn(L, Hq, p, 128, device="cuda").bfloat16(); kp = torch.randn(L, H, p, 128, device="cuda").bfloat16()
    posn = torch.arange(start, start + B, dtype=torch.int32, device="cuda"); start += B
    print("step", step, "a.off", a.head_off[0].tolist(), "a.len", a.head_len[0].tolist(), flush=True)
    gpu.append_to_cache(a, kn, vn, posn, ctx=ctx); torch.cuda.synchronize()
    try: ctx.poll_error()
    except Exception as e: print("after append", e); break
    print("  after append len", a.head_len[0].tolist())
    scores = torch.zeros(a.rows, dtype=torch.float32, device="cuda")
    evict_step(a, b, q, kp, [M] * L, mode="tc_bf16", slack=B, n_max_per_head=M + B, scores=scores, ctx=ctx)
    torch.cuda.synchronize()
    try: ctx.poll_error()
    except Exception as e: print("after step", e); 
    print("  out off", b.head_off[0].tolist(), "len", b.head_len[0].tolist(), flush=True)
    a, b = b, a
