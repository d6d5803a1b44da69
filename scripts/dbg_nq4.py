import sys; sys.path.insert(0, '.')
import numpy as np, torch, time
import paper_2509_17396_b200 as gpu
from tests.helpers import bf16_round, random_layer
L, Hq, H, p, n = int(sys.argv[1]), int(sys.argv[2]), 8, 128, int(sys.argv[3])
c = gpu.EpisodeCache(L, H, 128, [n * H] * L, torch.bfloat16, "cuda")
c.set_regions(n)
c.head_len.fill_(n)
c.k.normal_(); c.v.normal_()
q = torch.randn(L, Hq, p, 128, device="cuda").bfloat16(); kp = torch.randn(L, H, p, 128, device="cuda").bfloat16()
for it in range(int(sys.argv[4])):
    t = time.time()
    sc = gpu.score_with_prompt(c, q, kp, "max", mode="tc_bf16")
    torch.cuda.synchronize()
    print("ok", it, round(time.time() - t, 4), flush=True)
