timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
for g in 28 0; do timeout 200 python bench.py --steps 300 --warmup 5 --no-e2e --no-cpu-baseline --layer-group $g > gpurun_out/sweep.json 2>gpurun_out/sweep.err; python -c "
import json; d=json.load(open('gpurun_out/sweep.json')); k=d['kernels']
print('g $g', round(d['ms_per_step'],4), {n: round(v['ms_per_step'],4) for n,v in k.items()})" || tail -3 gpurun_out/sweep.err; done
