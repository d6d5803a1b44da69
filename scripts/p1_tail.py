"""Per-CTA timing of the P1 (STATS) pass from an EPK_P1_PROF library variant:
reads the P1GT lines (CTA, globaltimer begin/end, SM, jobs, wait cycles) that
the variant prints and summarises the spread of CTA end times per launch."""
import re
import sys
import statistics

launches, cur = [], []
for line in open(sys.argv[1]):
    m = re.match(r"P1GT (\d+) (\d+) (\d+) (\d+) (\d+) (\d+) (\d+) (\d+) (\d+)", line)
    if not m:
        continue
    b, g0, g1, sm, jobs, wait, tot, i0, i1 = map(int, m.groups())
    if cur and any(x[0] == b for x in cur):
        launches.append(cur)
        cur = []
    cur.append((b, g0, g1, sm, jobs, wait, tot, i0, i1))
if cur:
    launches.append(cur)
for li, L in enumerate(launches[-3:]):
    t0 = min(x[1] for x in L)
    begs = sorted((x[1] - t0) / 1e3 for x in L)
    ends = sorted((x[2] - t0) / 1e3 for x in L)
    durs = sorted((x[2] - x[1]) / 1e3 for x in L)
    waits = sorted(x[5] for x in L)
    print(f"launch {li}: CTAs {len(L)}  begin us min/med/max {begs[0]:.1f}/{statistics.median(begs):.1f}/{begs[-1]:.1f}"
          f"  end us min/med/max {ends[0]:.1f}/{statistics.median(ends):.1f}/{ends[-1]:.1f}"
          f"  dur us min/med/max {durs[0]:.1f}/{statistics.median(durs):.1f}/{durs[-1]:.1f}"
          f"  wait cyc med {statistics.median(waits)}"
          f"  SM clock GHz med {statistics.median(x[6] / max(1, x[2] - x[1]) for x in L):.3f}")
    slow = sorted(L, key=lambda x: x[2])[-5:]
    print("  last-ending CTAs (cta, sm, begin us, dur us, tiles):",
          [(x[0], x[3], round((x[1] - t0) / 1e3, 1), round((x[2] - x[1]) / 1e3, 1), x[8] - x[7]) for x in slow])
