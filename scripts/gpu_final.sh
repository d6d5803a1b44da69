#!/bin/bash
# end-of-round sequence: pytest -m gpu, smoke(), the default bench line (driver
# flags), the other configs' lines, the reference arm, ncu evidence, sanitizers
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/smi.txt 2>&1; cat MEASURED_PEAKS.json > gpurun_out/peaks.json 2>/dev/null
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
for cfg in cfg3 cfg4 cfg5 cfg1; do
  timeout 900 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --no-exact > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err
done
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
[ -n "$NO_NCU" ] || bash scripts/ncu_r02b.sh > gpurun_out/ncu_run.log 2>&1
[ -n "$NO_SAN" ] || bash scripts/sanitize.sh > gpurun_out/sanitize.log 2>&1
grep -E "passed|failed|FAILED|rc=" gpurun_out/gpu_tests.log | tail -5; tail -2 gpurun_out/smoke.log; tail -1 gpurun_out/bench.err
cat gpurun_out/sanitize.log 2>/dev/null | grep -E "==|SUMMARY"
for f in gpurun_out/bench.json gpurun_out/bench_cfg*.json gpurun_out/bench_ref.json; do
  python -c "
import json,sys
try:
    d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d.get('ms_per_step'), d.get('value'), (d.get('step_roofline') or {}).get('frac'), (d.get('roofline') or {}).get('frac'))
except Exception as e: print('$f', 'ERR', e)"
done
