"""Summarise a CTA-0 timeline written by the scorer under EPK_TC_TRACE."""
import sys
import numpy as np
a = np.fromfile(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/p2_trace.bin", dtype=np.uint64)[1:]
R = 60000
names = {1: "prod wait k_empty", 2: "prod got k_empty", 3: "mma wait k_full", 4: "mma got k_full", 5: "mma wait t_empty",
         6: "mma got t_empty", 7: "mma issued job", 8: "epi wait t_full", 9: "epi got t_full", 10: "epi ld+math 64",
         11: "epi tile done"}
allt = []
for role in range(3):
    r = a[role * R:(role + 1) * R]
    r = r[r != 0]
    allt.append((role, (r >> 56).astype(int), (r & 0xFFFFFFFFFFFFFF).astype(np.int64)))
t0 = min(t.min() for _, _, t in allt)
for role, ev, t in allt:
    t = t - t0
    print("role", role, "records", len(t), "span", t.max() - t.min())
    for w0, w1 in ((1, 2), (3, 4), (5, 6), (8, 9)):
        s, e = t[ev == w0], t[ev == w1]
        m = min(len(s), len(e))
        if m:
            d = e[:m] - s[:m]
            print(f"   {names[w0]:20s} n={m:5d} total={d.sum():9d} mean={d.mean():8.1f}")
    if role == 1:
        iss = t[ev == 7]
        got = t[ev == 6]
        m = min(len(iss), len(got))
        print("   mma jobs", len(iss), "mean gap", np.diff(iss).mean(), " got t_empty->issued mean", (iss[:m] - got[:m]).mean())
m = sorted((tt - t0, role, e_) for role, ev, t in allt for e_, tt in zip(ev, t))
for tt, role, e_ in m[300:340]:
    print(f"{tt:9d} r{role} {names.get(e_, e_)}")
