"""Prints the headline metrics of ncu reports (ncu -i ... --page raw --csv)."""
import csv, subprocess, sys

WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'launch__grid_size', 'launch__block_size',
        'launch__registers_per_thread', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'lts__t_bytes.sum', 'sm__cycles_active.avg']
STALL = 'smsp__average_warps_issue_stalled_'


def summary(path):
    out = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, u = r[0], r[1]
    res = []
    for row in r[2:]:
        d = {}
        for w in WANT:
            if w in h:
                d[w] = (row[h.index(w)], u[h.index(w)])
        st = [(float(row[i]), h[i][len(STALL):].replace('_per_issue_active.ratio', ''))
              for i in range(len(h)) if h[i].startswith(STALL) and h[i].endswith('per_issue_active.ratio')
              and row[i] not in ('', 'n/a')]
        st.sort(reverse=True)
        d['top_stalls'] = [(n, round(v, 3)) for v, n in st[:6]]
        res.append((row[h.index('Kernel Name')] if 'Kernel Name' in h else '?', d))
    return res


if __name__ == '__main__':
    for p in sys.argv[1:]:
        for name, d in summary(p):
            print('==', p, name[:60])
            for k, v in d.items():
                print('  ', k, v)
