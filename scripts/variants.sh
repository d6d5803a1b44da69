# run scripts/bench_brief.sh against each prebuilt library variant in _variants/
cp paper_2509_17396_b200/libepk.so /tmp/libepk_orig.so
for v in ${VARIANTS:-_variants/*.so}; do
  cp "$v" paper_2509_17396_b200/libepk.so
  echo "== $v"; REPS=${REPS:-2} bash scripts/bench_brief.sh "$@"
done
cp /tmp/libepk_orig.so paper_2509_17396_b200/libepk.so
