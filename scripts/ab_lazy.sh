#!/bin/bash
# A/B of P1 epilogue variants (_variants/*.so): parity of the tensor-core scorer under each, then the brief bench per variant
mkdir -p gpurun_out
cp paper_2509_17396_b200/libepk.so /tmp/libepk_orig.so
for v in ${TVARIANTS:-}; do
  cp _variants/$v.so paper_2509_17396_b200/libepk.so
  timeout 600 python -m pytest -q -m gpu tests/test_gpu_score_tc.py -x > gpurun_out/ab_tests_$v.log 2>&1; echo "$v tests rc=$?" >> gpurun_out/ab_tests.log
done
cp /tmp/libepk_orig.so paper_2509_17396_b200/libepk.so
VARIANTS="$VARIANTS" REPS=${REPS:-2} bash scripts/variants.sh > gpurun_out/ab.log 2>&1
cat gpurun_out/ab_tests.log; cat gpurun_out/ab.log
