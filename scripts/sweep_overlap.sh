#!/bin/bash
# SM-partition / layer-group sweep of the default step (bench.py, cfg2)
mkdir -p gpurun_out; out=gpurun_out/sweep.txt; : > $out
run() {  # label, env..., -- bench args
  local label=$1; shift
  local envs=(); while [ "$1" != "--" ]; do envs+=("$1"); shift; done; shift
  env "${envs[@]}" timeout 300 python bench.py --steps 200 --warmup 10 --no-e2e --no-cpu-baseline "$@" > /tmp/b.json 2>/tmp/b.err
  python - "$label" <<'PY' >> gpurun_out/sweep.txt
import json, sys
try:
    d = json.loads(open('/tmp/b.json').read().strip().splitlines()[-1])
    k = d["kernels"]
    print(f"{sys.argv[1]:40s} {d['ms_per_step']:.4f} ms/step  " + "  ".join(f"{n} {v['ms_per_step']:.3f}" for n, v in k.items()))
except Exception as e:
    print(sys.argv[1], "FAILED", open('/tmp/b.err').read()[-500:])
PY
}
run "default" X=1 --
run "g14" X=1 -- --layer-group 14
run "g7" X=1 -- --layer-group 7
run "g4" X=1 -- --layer-group 4
for S in 24 32 40; do
  for g in 4 7; do
    run "split S=$S g$g" EPK_GATHER_SMS=$S EPK_GATHER_CTAS=$S EPK_GATHER_THREADS=512 EPK_GATHER_SMEM_KB=120 -- --layer-group $g
  done
done
run "corun148 g4" EPK_GATHER_CTAS=148 EPK_GATHER_THREADS=128 -- --layer-group 4
run "corun296 g7" EPK_GATHER_CTAS=296 EPK_GATHER_THREADS=128 -- --layer-group 7
cat $out
