#!/bin/bash
# quick state check: pytest -m gpu, smoke(), the default bench line
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
grep -E "passed|failed|FAILED|rc=" gpurun_out/gpu_tests.log | tail -8; tail -2 gpurun_out/smoke.log; tail -3 gpurun_out/bench.err
python -c "
import json
d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1])
print({k:d.get(k) for k in ('value','ms_per_step','clocks','roofline','step_roofline','kernels')})
"
