import sys, os, time; sys.path.insert(0, '.')
import torch
import paper_2509_17396_b200 as epk
from paper_2509_17396_b200.step import StepPlan, evict_step
import bench
c = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg4"]
dev = torch.device("cuda", 0)
ctx = epk.default_context(0)
ctx.profile(True)
caches, qs, kps, out = bench.make_inputs(epk, torch, c, 2, dev, 1)
n_h, live, keep = bench.step_sizes(c)
budgets = [c["M"]] * c["L"]
for i in range(4):
    r = i % 2
    evict_step(caches[r], out, qs[r], kps[r], budgets, mode="tc_bf16", slack=c["block"], n_max_per_head=n_h, ctx=ctx)
    t = time.time()
    torch.cuda.synchronize()
    print("step", i, "ok", time.time() - t, [n for n, _ in ctx.profile_records()][-7:], flush=True)
