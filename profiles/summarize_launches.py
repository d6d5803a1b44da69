"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
per-kernel mean durations and the share of our kernels in one step."""
import collections
import csv
import sys


def main(path, out):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.reader(lines[start:]))
    h = rows[0]
    i_name, i_val = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[1:]:
        n = r[i_name].split("(")[0].replace("void ", "").replace("epk::", "")
        n = n.replace("tc_score_kernel<0>", "tc_score_kernel<P1>").replace("tc_score_kernel<1>", "tc_score_kernel<P2>")
        agg.setdefault(n, []).append(float(r[i_val].replace(",", "")))
    ours = {n: v for n, v in agg.items() if n.startswith(("tc_", "select", "compact", "f32_", "append", "step_"))}
    tot = sum(sum(v) / len(v) for v in ours.values())
    with open(out, "w") as f:
        f.write(f"# source: {path}\n# ncu --metrics gpu__time_duration.sum --clock-control none: cold-cache, "
                "serialised; compare SHARES, not absolutes\n")
        f.write(f"{'kernel':32s} {'launches':>8s} {'mean_us':>10s} {'share_of_step':>14s}\n")
        for n, v in ours.items():
            m = sum(v) / len(v)
            f.write(f"{n:32s} {len(v):8d} {m / 1000:10.1f} {m / tot:14.3f}\n")
        f.write(f"{'step (sum of means)':32s} {'':8s} {tot / 1000:10.1f}\n")
    print(open(out).read())


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
