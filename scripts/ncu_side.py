"""One launch of every non-step kernel family at its SURVEY 8(d) size, for
`ncu --set full` (scripts/ncu_r02.sh): K5 pair + chain (cfg2 calibration,
EPK_K5_SERIAL=1 so the profiler's serialisation cannot starve the chain),
K4 assign / sums (2,048 x 1,024, k = 4), KeyDiff, the .epkv writer and
reader, append, score pooling (cfg2 step sizes)."""
import os
import sys
import tempfile

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_17396_b200 as epk  # noqa: E402

kf = torch.randn(28, 8, 32768, 128, device="cuda").bfloat16()
kb = (kf.float() + 0.3 * torch.randn_like(kf.float())).bfloat16()
epk.sensitivity_from_keys(kf, kb)
del kf, kb
rng = np.random.default_rng(0)
pts = rng.standard_normal((4, 1024))[rng.integers(0, 4, 2048)] + rng.standard_normal((2048, 1024))
epk.kmeans(pts, 4, 1, max_iters=2)
L, H, d, n = 28, 8, 128, 10240
c = epk.EpisodeCache(L, H, d, [H * (n + 2048)] * L, torch.bfloat16, "cuda")
c.set_regions(n + 2048)
c.head_len.fill_(n)
c.k.normal_()
c.v.normal_()
c.pos.copy_(torch.arange(c.rows, device="cuda", dtype=torch.int32) % (n + 2048))
epk.keydiff_scores(c)
epk.pool_scores(c, torch.rand(c.rows, device="cuda"), 7)
epk.append_to_cache(c, torch.randn(L, H, 2048, d, device="cuda").bfloat16(),
                    torch.randn(L, H, 2048, d, device="cuda").bfloat16(),
                    torch.arange(20000, 22048, device="cuda", dtype=torch.int32))
c.head_len.fill_(8192)
path = os.path.join(tempfile.mkdtemp(), "ep.epkv")
epk.persist(c, path)
epk.retrieve(path)
torch.cuda.synchronize()
print("ncu side pass done")
