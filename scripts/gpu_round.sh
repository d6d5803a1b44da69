#!/bin/bash
# the round-end sequence: pytest -m gpu, smoke(), default bench, the reference arm, extra bench lines, retrieve timing
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/smi.txt 2>&1; cat MEASURED_PEAKS.json > gpurun_out/peaks.json 2>/dev/null
timeout 1800 python -m pytest tests -q -m gpu -s > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
for cfg in cfg4 cfg5 cfg1; do
  timeout 900 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --no-exact > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err
done
timeout 600 python scripts/time_retrieve.py > gpurun_out/retrieve.json 2>&1
grep -E "passed|failed|FAILED|rc=" gpurun_out/gpu_tests.log | tail -5; cat gpurun_out/smoke.log | tail -2; tail -1 gpurun_out/bench.err
