# P1 exp2 split sweep: EPK_TC_POLY = pairs of every 4 whose exp2 runs on the FMA pipe
for poly in 0 1 2 0; do
  echo "POLY=$poly"
  EPK_TC_POLY=$poly REPS=1 bash scripts/bench_brief.sh --sustained-steps 0 --no-exact
done
