cp paper_2509_17396_b200/libepk.so /tmp/libepk_orig.so
for v in default _variants/EPK_XP_NOEXP.so _variants/EPK_XP_NOEXP_NOMMA.so; do
  [ $v != default ] && cp $v paper_2509_17396_b200/libepk.so
  for kb in 200 226; do
    echo "== $v smem $kb"; EPK_TC_VERBOSE=1 EPK_TC_SMEM_KB=$kb timeout 300 python scripts/xp_time.py 20 2>&1 | grep -E "^P1|^step" | tail -2
  done
done
cp /tmp/libepk_orig.so paper_2509_17396_b200/libepk.so
