#!/bin/bash
mkdir -p gpurun_out; out=gpurun_out/sweep2.txt; : > $out
run() {
  local label=$1; shift
  timeout 300 python bench.py --steps 200 --warmup 10 --no-e2e --no-cpu-baseline "$@" > /tmp/b.json 2>/tmp/b.err
  python - "$label" <<'PY' >> $out
import json, sys
try:
    d = json.loads(open('/tmp/b.json').read().strip().splitlines()[-1])
    k = d["kernels"]
    print(f"{sys.argv[1]:30s} {d['ms_per_step']:.4f} ms/step  " + "  ".join(f"{n} {v['ms_per_step']:.3f}" for n, v in k.items()))
except Exception as e:
    print(sys.argv[1], "FAILED", open('/tmp/b.err').read()[-500:])
PY
}
run default
run "g4 serial" --layer-group 4 --no-overlap
run "g7 serial" --layer-group 7 --no-overlap
run "g14 serial" --layer-group 14 --no-overlap
timeout 600 python scripts/time_k4k5.py > gpurun_out/k4k5.json 2>&1
timeout 600 python -m pytest tests -q -m gpu -k "kmeans or sensitiv or phase_a or hardening" > gpurun_out/t.log 2>&1; echo "rc=$?" >> gpurun_out/t.log
cat $out gpurun_out/k4k5.json; tail -3 gpurun_out/t.log
