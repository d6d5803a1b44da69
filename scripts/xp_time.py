"""Experiment timer: the cfg2 step's per-kernel times (live CUDA events,
ctx.profile) and the step time, IGNORING deferred device errors -- for
library variants built with experiment switches (EPK_XP_*) whose results are
deliberately wrong.  Usage: python scripts/xp_time.py [steps]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2509_17396_b200 as epk  # noqa: E402
from paper_2509_17396_b200.step import StepPlan, evict_step  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
c = bench.CONFIGS[os.environ.get("XP_CFG", "cfg2")]
dev = torch.device("cuda:0")
ctx = epk.default_context(0)
n_h, live, keep = bench.step_sizes(c)
caches, qs, kps, out = bench.make_inputs(epk, torch, c, 3, dev, 1234)
budgets = bench.layer_budgets(c)
plans = [StepPlan(caches[r], out, budgets) for r in range(3)]


def step(i):
    r = i % 3
    evict_step(caches[r], out, qs[r], kps[r], budgets, mode="tc_bf16", slack=c["block"], n_max_per_head=n_h,
               plan=plans[r], ctx=ctx)


def poll():
    try:
        ctx.poll_error()
    except Exception as e:  # noqa: BLE001
        return str(e)[:60]
    return ""


for i in range(5):
    step(i)
torch.cuda.synchronize()
err = poll()
s = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
time.sleep(0.2)
e0.record(s)
for i in range(steps):
    step(i)
e1.record(s)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
poll()
ctx.profile(True)
for i in range(steps):
    step(i)
recs = ctx.profile_records()
ctx.profile(False)
poll()
k = {}
for name, kms in recs:
    k[name] = k.get(name, 0.0) + kms / steps
print(f"step {ms:.4f} ms  " + "  ".join(f"{n} {v:.4f}" for n, v in k.items()) + (f"  [err: {err}]" if err else ""))
