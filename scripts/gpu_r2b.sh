#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -s -x > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
for v in paper_2509_17396_b200/libepk.so _variants/libepk_e8m2.so _variants/libepk_e8m1.so; do
  timeout 300 python scripts/probes/corun.py $v >> gpurun_out/corun.txt 2>&1
done
grep -E "passed|failed|error|cfg|tie|rc=" gpurun_out/gpu_tests.log | tail -30; cat gpurun_out/corun.txt
