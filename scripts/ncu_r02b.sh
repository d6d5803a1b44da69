#!/bin/bash
# round-2 (final build) ncu evidence for the cfg2 step: the launch list
# (gpu__time_duration of every launch) and one --set full capture of each step
# kernel: P1 (tc_score_kernel<0>), the lse-bias merge, P2 (tc_score_kernel<1>),
# the threshold select (+ compaction plan) and the gather
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-exact --sustained-steps 0"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02b.csv $B > /dev/null 2>&1
for k in tc_score_kernelILi0:p1 tc_bias_kernel:bias tc_score_kernelILi1:p2 select_threshold_kernel:sel compact_gather:gather; do
  IFS=: read pat nm <<< "$k"
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k "regex:$pat" -s 3 -c 1 \
    -o gpurun_out/r02b_$nm $B > gpurun_out/ncu_$nm.log 2>&1
done
ls gpurun_out/r02b_*.ncu-rep
