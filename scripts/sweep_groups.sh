# layer-group / overlap sweep of the cfg2 step (ms per step, per-kernel ms)
for opt in "--layer-group 28 --no-overlap" "--layer-group 14" "--layer-group 7" "--layer-group 4" "--layer-group 2" "--layer-group 7 --no-overlap"; do
  timeout 200 python bench.py --steps 300 --warmup 5 --no-e2e --no-cpu-baseline $opt > gpurun_out/sweep.json 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/sweep.json')); k=d['kernels']
print('$opt', round(d['ms_per_step'],4), {n: round(v['ms_per_step'],4) for n,v in k.items()})" || tail -5 gpurun_out/sweep.json
done
