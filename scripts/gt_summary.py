"""Summarise P1GT/P2GT lines (EPK_P1_PROF builds): per launch, kernel-entry
spread, epilogue start and end distribution relative to the first CTA entry."""
import sys
from collections import defaultdict
runs = defaultdict(list)
for line in open(sys.argv[1]):
    if "GT " not in line or not line.startswith("P"):
        continue
    f = line.split()
    kind = f[0]
    cta, gb, ge, k0 = int(f[1]), int(f[2]), int(f[3]), int(f[10])
    runs[kind].append((cta, k0, gb, ge))
for kind, rows in runs.items():
    n = len(rows) // 148
    for i in range(n):
        r = rows[i * 148:(i + 1) * 148]
        t0 = min(x[1] for x in r)
        k0 = sorted((x[1] - t0) / 1e3 for x in r)
        gb = sorted((x[2] - t0) / 1e3 for x in r)
        ge = sorted((x[3] - t0) / 1e3 for x in r)
        print(f"{kind} launch {i}: entry max {k0[-1]:.1f} us, epi start med {gb[74]:.1f} max {gb[-1]:.1f}, "
              f"epi end min {ge[0]:.1f} med {ge[74]:.1f} max {ge[-1]:.1f} us")
