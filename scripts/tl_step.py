"""Critical path of one cfg2 step from an EPK_TIMELINE library variant
(-DEPK_TIMELINE): every warp of P1 / bias / P2 / select / gather records
globaltimer at entry, after griddepcontrol.wait, and at exit; this prints per
launch the first entry, first / last go, median / last end (us from the
step's first entry).  Usage: python scripts/tl_step.py (with the variant
library in place, see scripts/tl_run.sh)"""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2509_17396_b200 as epk  # noqa: E402
from paper_2509_17396_b200 import _lib  # noqa: E402
from paper_2509_17396_b200.step import StepPlan, evict_step  # noqa: E402

c = bench.CONFIGS[os.environ.get("XP_CFG", "cfg2")]
dev = torch.device("cuda:0")
ctx = epk.default_context(0)
n_h, live, keep = bench.step_sizes(c)
caches, qs, kps, out = bench.make_inputs(epk, torch, c, 3, dev, 1234)
budgets = bench.layer_budgets(c)
plans = [StepPlan(caches[r], out, budgets) for r in range(3)]
lib = _lib.load()
f = lib.epk_debug_timeline
f.restype = ctypes.c_int
f.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int]
NAMES = {1: "p1", 2: "p2", 3: "bias", 4: "select", 5: "select", 6: "gather"}
for i in range(8):
    if i == 6:
        f(1, None, 0)
    evict_step(caches[i % 3], out, qs[i % 3], kps[i % 3], budgets, mode="tc_bf16", slack=c["block"],
               n_max_per_head=n_h, plan=plans[i % 3], ctx=ctx)
torch.cuda.synchronize()
buf = np.zeros((1 << 19, 4), dtype=np.uint64)
n = f(1, buf.ctypes.data, buf.shape[0])
rec = buf[:n]
kid = (rec[:, 0] >> np.uint64(32)).astype(int)
t0 = None
order = ["p1", "bias", "p2", "select", "gather"]
# records hold two steps (6 and 7): split each kernel's records by entry time
for step in (0, 1):
    rows = {}
    for name in order:
        ids = [k for k, v in NAMES.items() if v == name]
        m = np.isin(kid, ids)
        r = rec[m]
        if len(r) == 0:
            continue
        ent = r[:, 1].astype(np.int64)
        cut = np.sort(ent)
        # the two launches of a kernel: split at the largest gap in entry times
        gaps = np.diff(cut)
        split = cut[int(np.argmax(gaps)) + 1] if len(gaps) else cut[0] + 1
        sel = ent < split if step == 0 else ent >= split
        rows[name] = r[sel].astype(np.int64)
    t0 = min(v[:, 1].min() for v in rows.values())
    if step == 1:
        print(f"-- gap: step 1 first entry - step 0 last end = {(t0 - s0_end) / 1e3:.2f} us")
    s0_end = max(v[:, 3].max() for v in rows.values())
    print(f"-- step {step}")
    prev = None
    for name in order:
        if name not in rows:
            continue
        r = rows[name]
        ent, go, end = r[:, 1] - t0, r[:, 2] - t0, r[:, 3] - t0
        gap = "" if prev is None else f"  go-after-prev-end {(go.min() - prev) / 1e3:7.2f}"
        print(f"{name:7s} entry {ent.min() / 1e3:8.2f}  go {go.min() / 1e3:8.2f}..{go.max() / 1e3:8.2f}  "
              f"end med {np.median(end) / 1e3:8.2f} max {end.max() / 1e3:8.2f} us{gap}")
        prev = end.max()
    print(f"step span {prev / 1e3:.2f} us")
    # select sub-phases (ids 7..12: after the histograms, after the key loads,
    # slice done, resolve done, candidates added, scan done): median of
    # (mark - go) over the warps of this step's select launch
    go_sel = rows["select"][:, 2].min() if "select" in rows else None
    for mid, what in ((7, "hist"), (8, "keys"), (9, "slice"), (10, "resolve"), (11, "cand add"), (12, "scan")):
        r = rec[kid == mid].astype(np.int64)
        if len(r) and go_sel is not None:
            r = r[(r[:, 2] >= go_sel) & (r[:, 2] < go_sel + 200000)]
            if len(r):
                d = (r[:, 3] - r[:, 2]) / 1e3
                print(f"   select {what:8s} mark-go med {np.median(d):6.2f} max {d.max():6.2f} us (n={len(r)})")
