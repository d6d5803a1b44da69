"""Toy-shape pass over every kernel family for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck): the tensor-core scorer
(P1 + P2 with fused histograms), threshold select, count / plan / gather,
generic select, the fp32 parity scorer, append, pooling, KeyDiff, the .epkv
writer, K4 (sharded chain) and K5 (pair + chain kernels)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_17396_b200 as epk  # noqa: E402
from paper_2509_17396_b200.context import Context  # noqa: E402
from paper_2509_17396_b200.step import evict_step  # noqa: E402

torch.manual_seed(0)
rng = np.random.default_rng(0)
L, H, Hq, p, d, slack, M = 2, 4, 12, 16, 128, 8, 60
for dtype, mode in ((torch.bfloat16, "tc_bf16"), (torch.float32, "exact_f32")):
    counts = [[100, 0, 37, 130], [70, 70, 70, 70]]
    per = []
    for c in counts:
        n = sum(c)
        pos = np.concatenate([np.sort(rng.choice(300, x, replace=False)) for x in c]).astype(np.int64)
        per.append((np.array(c), pos, rng.standard_normal((n, d)).astype(np.float32),
                    rng.standard_normal((n, d)).astype(np.float32)))
    cap = [sum(c) + slack * H + 16 for c in counts]
    cin = epk.EpisodeCache(L, H, d, cap, dtype, "cuda")
    cin.load_layers(per, slack=slack)
    cout = epk.EpisodeCache(L, H, d, cap, dtype, "cuda")
    q = torch.randn(L, Hq, p, d, device="cuda").to(dtype)
    kp = torch.randn(L, H, p, d, device="cuda").to(dtype)
    sc = torch.zeros(cin.rows, device="cuda")
    evict_step(cin, cout, q, kp, [M] * L, mode=mode, slack=slack, scores=sc)
    keep = epk.select_pooled(cin, sc, [M] * L, pinned={int(per[0][1][0])})
    epk.compact(cin, keep, cout, slack=slack)
    epk.append_to_cache(cout, torch.randn(L, H, 4, d, device="cuda").to(dtype),
                        torch.randn(L, H, 4, d, device="cuda").to(dtype),
                        torch.arange(400, 404, device="cuda", dtype=torch.int32), slack=slack)
    if mode == "tc_bf16":
        epk.pool_scores(cin, sc, 5)
        epk.keydiff_scores(cin)
        epk.default_context(0).set_option(layer_group=1, overlap=True)
        evict_step(cin, cout, q, kp, [M] * L, mode=mode, slack=slack, scores=sc)
        epk.default_context(0).set_option(layer_group=0)
    torch.cuda.synchronize()
    epk.default_context(0).poll_error()
kf = torch.randn(2, 2, 300, 64, device="cuda").bfloat16()
kb = (kf.float() + 0.3 * torch.randn_like(kf.float())).bfloat16()
epk.sensitivity_from_keys(kf, kb)
pts = rng.standard_normal((90, 16))
ctxs = [Context(0) for _ in range(3)]
epk.kmeans_multi_device(pts, 4, 1, contexts=ctxs)
epk.kmeans(pts, 4, 1)
torch.cuda.synchronize()
print("sanitize pass done")
