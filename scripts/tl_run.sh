# one-step critical path from the EPK_TIMELINE variant (scripts/tl_step.py)
mkdir -p gpurun_out
cp paper_2509_17396_b200/libepk.so /tmp/libepk_orig.so
cp ${1:-_variants/tl.so} paper_2509_17396_b200/libepk.so
timeout 300 python scripts/tl_step.py > gpurun_out/tl.out 2>&1
cp /tmp/libepk_orig.so paper_2509_17396_b200/libepk.so
cat gpurun_out/tl.out | tail -16
