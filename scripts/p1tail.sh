# P1 per-CTA timing and per-role wait cycles from the EPK_P1_PROF variant (scripts/p1_tail.py)
mkdir -p gpurun_out
cp paper_2509_17396_b200/libepk.so /tmp/libepk_orig.so
cp ${1:-_variants/p1prof.so} paper_2509_17396_b200/libepk.so
timeout 300 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-exact --sustained-steps 0 > gpurun_out/p1prof.out 2> gpurun_out/p1prof.err
cp /tmp/libepk_orig.so paper_2509_17396_b200/libepk.so
python scripts/p1_tail.py gpurun_out/p1prof.out
grep "P1PROF cta 0 " gpurun_out/p1prof.out | tail -16
