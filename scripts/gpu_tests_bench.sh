#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 900 python bench.py --config cfg3 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
grep -E "passed|failed|FAILED|rc=" gpurun_out/gpu_tests.log | tail -8; tail -3 gpurun_out/bench.err; python -c "
import json
for f in ['gpurun_out/bench.json','gpurun_out/bench_cfg3.json','gpurun_out/bench_ref.json']:
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, {k:d.get(k) for k in ('value','ms_per_step','steps','warmup')}, 'sus', (d.get('sustained') or {}).get('ms_per_step'), 'exact', (d.get('exact_f32') or {}).get('ms_per_step'), 'cpu', d.get('cpu_baseline'), 'phase_a', d.get('phase_a'), 'roof', d.get('roofline'))
    except Exception as e: print(f, 'ERR', e)
"
