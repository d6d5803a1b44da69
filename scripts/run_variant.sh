# run bench.py once against a prebuilt library variant: run_variant.sh <variant.so> [bench args...]
v=$1; shift
cp paper_2509_17396_b200/libepk.so /tmp/libepk_orig.so
cp "$v" paper_2509_17396_b200/libepk.so
timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-exact --sustained-steps 0 "$@" > gpurun_out/variant.out 2> gpurun_out/variant.err
echo "rc=$?"
cp /tmp/libepk_orig.so paper_2509_17396_b200/libepk.so
