for ks in 2 3 4; do
  EPK_TC_VERBOSE=1 EPK_P2_KSTAGES=$ks EPK_P1_KSTAGES=$ks timeout 200 python bench.py --steps 200 --warmup 5 --no-e2e --no-cpu-baseline --layer-group 28 > gpurun_out/sw.json 2> gpurun_out/sw.err
  head -2 gpurun_out/sw.err
  python -c "
import json; d=json.load(open('gpurun_out/sw.json')); k=d['kernels']
print('kstages=$ks', round(d['ms_per_step'],4), {n: round(v['ms_per_step'],4) for n,v in k.items() if n.startswith('p')})"
done
