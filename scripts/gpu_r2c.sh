#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/corun.txt
for v in paper_2509_17396_b200/libepk.so _variants/libepk_e8m2.so _variants/libepk_co100.so _variants/libepk_co100_e8m2.so; do
  timeout 300 python scripts/probes/corun.py $v >> gpurun_out/corun.txt 2>&1
done
timeout 1500 python -m pytest tests -q -m gpu -s > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
cat gpurun_out/corun.txt; grep -E "passed|failed|FAILED|Error|cfg|tie|rc=" gpurun_out/gpu_tests.log | tail -30
