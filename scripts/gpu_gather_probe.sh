#!/bin/bash
# round-2 first call: baseline tests + bench + the gather-per-SM probe
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/smi.txt 2>&1; nproc >> gpurun_out/smi.txt; lscpu | grep "Model name" >> gpurun_out/smi.txt
timeout 300 ./scripts/probes/gather_sm > gpurun_out/gather_sm.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 50 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
tail -3 gpurun_out/gpu_tests.log; cat gpurun_out/gather_sm.txt; head -c 1500 gpurun_out/bench.json
