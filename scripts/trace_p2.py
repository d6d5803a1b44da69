"""Diagnostic: run one bench step with EPK_TC_TRACE and summarise CTA 0's P2 timeline."""
import os, subprocess, sys
import numpy as np
path = "gpurun_out/p2_trace.bin"
env = dict(os.environ, EPK_TC_TRACE=path)
subprocess.run([sys.executable, "bench.py", "--steps", "3", "--warmup", "1", "--no-e2e", "--no-cpu-baseline",
                "--layer-group", "28"], env=env, check=True, stdout=subprocess.DEVNULL)
a = np.fromfile(path, dtype=np.uint64)[1:]
r = a[a != 0]
n = len(r)
ev = (r >> 56).astype(int); t = (r & 0xFFFFFFFFFFFFFF).astype(np.int64)
t = t - t.min()
names = {1: "prod wait k_empty", 2: "prod got k_empty", 3: "mma wait k_full", 4: "mma got k_full", 5: "mma wait t_empty",
         6: "mma got t_empty", 7: "mma issued job", 8: "epi wait t_full", 9: "epi got t_full", 10: "epi ld+math 64",
         11: "epi tile done"}
order = np.argsort(t, kind="stable")
ev, role, t = ev[order], role[order], t[order]
print("records", n, "span cycles", t.max())
# time spent waiting per wait type
for w0, w1 in ((1, 2), (3, 4), (5, 6), (8, 9)):
    starts = t[ev == w0]; ends = t[ev == w1]
    m = min(len(starts), len(ends))
    d = ends[:m] - starts[:m]
    print(f"{names[w0]:20s} n={m:6d} total={d.sum():10d} cyc  mean={d.mean() if m else 0:8.1f}  max={d.max() if m else 0}")
iss = t[ev == 7]
print("mma jobs", len(iss), "mean gap between job issues", np.diff(iss).mean() if len(iss) > 1 else 0)
print("first 60 events:")
for i in range(min(60, len(t))):
    print(f"  {t[i]:9d} {names.get(ev[i], ev[i])}")
