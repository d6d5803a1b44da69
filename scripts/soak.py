"""Soak / leak check of the throughput path on the box:

1. cfg2 block steps back to back for SOAK_SECS (default 60 s) on three rotating
   resident caches (as bench.py), polling the deferred device error every
   1,000 steps; reports steps, ms per step over the whole run, and that the
   final step's kept counts are the budgets.
2. 200 rounds of context create -> one small tensor-core step -> destroy
   through the C ABI, checking that the device's free memory does not drift.
Usage: python scripts/soak.py"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2509_17396_b200 as epk  # noqa: E402
from paper_2509_17396_b200.context import Context  # noqa: E402
from paper_2509_17396_b200.step import StepPlan, evict_step  # noqa: E402

SECS = float(os.environ.get("SOAK_SECS", "60"))


def soak():
    c = bench.CONFIGS["cfg2"]
    dev = torch.device("cuda:0")
    ctx = epk.default_context(0)
    n_h, live, keep = bench.step_sizes(c)
    caches, qs, kps, out = bench.make_inputs(epk, torch, c, 3, dev, 1234)
    budgets = bench.layer_budgets(c)
    plans = [StepPlan(caches[r], out, budgets) for r in range(3)]
    kept = torch.zeros(c["L"], dtype=torch.int32, device=dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.time()
    ev0.record()
    i = 0
    while time.time() - t0 < SECS:
        for _ in range(1000):
            r = i % 3
            evict_step(caches[r], out, qs[r], kps[r], budgets, mode="tc_bf16", slack=c["block"],
                       n_max_per_head=n_h, plan=plans[r], kept_per_layer=kept, ctx=ctx)
            i += 1
        ctx.poll_error()  # synchronises; raises on any deferred device error
    ev1.record()
    torch.cuda.synchronize()
    ctx.poll_error()
    ms = ev0.elapsed_time(ev1) / i
    ok = kept.cpu().tolist() == [c["H"] * b for b in budgets]
    return {"steps": i, "wall_s": round(time.time() - t0, 1), "ms_per_step": round(ms, 4), "kept_ok": ok}


def leak():
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    free0, _ = torch.cuda.mem_get_info(0)
    rng = np.random.default_rng(0)
    L, Hq, H, d, p = 2, 6, 2, 128, 16
    counts = [300, 170]
    drift = []
    for it in range(200):
        ctx = Context(0)
        cin = epk.EpisodeCache(L, H, d, [sum(counts) + 64] * L, torch.bfloat16, "cuda:0")
        ho = np.concatenate([[0], np.cumsum(counts)])
        layers = []
        for _ in range(L):
            pos = np.concatenate([np.arange(k) for k in counts])
            layers.append((np.diff(ho), pos, rng.standard_normal((ho[-1], d)), rng.standard_normal((ho[-1], d))))
        cin.load_layers(layers)
        cout = epk.EpisodeCache(L, H, d, [sum(counts) + 64] * L, torch.bfloat16, "cuda:0")
        q = torch.randn(L, Hq, p, d, device="cuda:0").bfloat16()
        kp = torch.randn(L, H, p, d, device="cuda:0").bfloat16()
        evict_step(cin, cout, q, kp, [100] * L, mode="tc_bf16", slack=16, ctx=ctx)
        ctx.synchronize()
        ctx.poll_error()
        ctx.close()
        del cin, cout, q, kp
        if it % 50 == 49:
            torch.cuda.synchronize()
            torch.cuda.empty_cache()
            drift.append((free0 - torch.cuda.mem_get_info(0)[0]) / 2**20)
    return {"rounds": 200, "free_mem_drift_mib_every_50": [round(x, 1) for x in drift]}


if __name__ == "__main__":
    res = {"soak_cfg2": soak(), "context_churn": leak()}
    print(json.dumps(res))
