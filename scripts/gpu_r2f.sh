#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python scripts/time_k4k5.py > gpurun_out/k4k5.json 2>&1
tail -30 gpurun_out/gpu_tests.log | grep -v "^\.\.\.\.\.\.\.\.\.\.\.\.\.\.\.\.\.\.\.\." ; cat gpurun_out/k4k5.json
