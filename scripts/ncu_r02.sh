#!/bin/bash
# round-2 ncu evidence: launch list of the cfg2 step, --set full of every
# step kernel and of the side kernels (K4, K5, KeyDiff, store, append, pool)
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-exact --sustained-steps 0"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02.csv $B > /dev/null 2>&1
for k in tc_score_kernel:3:p1 tc_score_kernel:4:p2 select_threshold_kernel:1:sel compact_count_kernel:1:count compact_plan_kernel:1:plan compact_gather:1:gather; do
  IFS=: read pat skip nm <<< "$k"
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$pat" -s $skip -c 1 -o gpurun_out/r02_$nm $B > gpurun_out/ncu_$nm.log 2>&1
done
for k in cosine_pair cosine_chain km_dist km_sums keydiff_anchor keydiff_score epkv_write epkv_read append_copy pool_scores; do
  EPK_K5_SERIAL=1 timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$k" -c 1 -o gpurun_out/r02_$k python scripts/ncu_side.py > gpurun_out/ncu_$k.log 2>&1
done
ls gpurun_out/*.ncu-rep | wc -l
