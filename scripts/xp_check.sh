# xp_check.sh <variant.so>... : per variant, the cfg2 step timing (xp_time.py) and the tensor-core parity tests
cp paper_2509_17396_b200/libepk.so /tmp/libepk_orig.so
echo "== default"; timeout 300 python scripts/xp_time.py 20 2>&1 | tail -1
for v in "$@"; do
  cp "$v" paper_2509_17396_b200/libepk.so
  echo "== $v"; timeout 300 python scripts/xp_time.py 20 2>&1 | tail -1; timeout 300 python scripts/xp_time.py 20 2>&1 | tail -1
  timeout 600 python -m pytest -q -x tests/test_gpu_score_tc.py tests/test_gpu_parity_scale.py 2>&1 | tail -1
done
cp /tmp/libepk_orig.so paper_2509_17396_b200/libepk.so
