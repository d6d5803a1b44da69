#!/bin/bash
# A/B of library variants with the driver's 20-step burst bench (0.2 % run-to-run spread):
# VARIANTS="a b ..." ROUNDS=3 bash scripts/ab_burst.sh  -> per variant the ms/step of every round
cp paper_2509_17396_b200/libepk.so /tmp/libepk_orig.so
for r in $(seq ${ROUNDS:-3}); do
  for v in $VARIANTS; do
    cp _variants/$v.so paper_2509_17396_b200/libepk.so
    ms=$(timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-exact --sustained-steps 0 --no-power-roofline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4))")
    echo "$v $ms"
  done
done
cp /tmp/libepk_orig.so paper_2509_17396_b200/libepk.so
