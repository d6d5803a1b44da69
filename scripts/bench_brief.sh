# brief cfg2 bench: ms/step and per-kernel ms per step, REPS times; extra args go to bench.py
REPS=${REPS:-2}
for i in $(seq $REPS); do
  timeout 200 python bench.py --steps 200 --warmup 5 --no-e2e --no-cpu-baseline "$@" > gpurun_out/brief.json 2> gpurun_out/brief.err
  python -c "
import json; d=json.loads(open('gpurun_out/brief.json').read().strip().splitlines()[-1]); k=d['kernels']
print(round(d['ms_per_step'],4), {n: round(v['ms_per_step'],4) for n,v in k.items()})" || tail -5 gpurun_out/brief.err
done
