timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for opt in "--layer-group 28 --no-overlap" "--layer-group 2 --no-overlap" "--layer-group 2" "--layer-group 1" "--layer-group 4"; do
  timeout 200 python bench.py --steps 300 --warmup 5 --no-e2e --no-cpu-baseline $opt > gpurun_out/sweep.json 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/sweep.json')); k=d['kernels']
print('$opt', round(d['ms_per_step'],4), {n: round(v['ms_per_step'],4) for n,v in k.items()})"
done
