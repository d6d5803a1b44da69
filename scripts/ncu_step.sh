# ncu captures of the cfg2 step kernels (1 GPU): launch list + full sets of the top kernels
OPT=${OPT:-}
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline $OPT"
[ -n "$LAUNCHES" ] && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > /dev/null 2>&1
for k in ${KERNELS:-tc_score_kernel:2:p1 tc_score_kernel:3:p2 select_threshold_kernel:1:sel compact_count_kernel:1:count compact_gather:1:gather}; do
  IFS=: read pat skip nm <<< "$k"
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$pat" -s $skip -c 1 -o gpurun_out/prof_$nm $B > gpurun_out/ncu_$nm.log 2>&1
done
ls -la gpurun_out
