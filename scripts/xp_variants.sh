# time the cfg2 step for the default library and each _variants/*.so given (xp_time.py; errors ignored)
cp paper_2509_17396_b200/libepk.so /tmp/libepk_orig.so
echo "== default"; timeout 300 python scripts/xp_time.py 20 2>&1 | tail -1
for v in "$@"; do
  cp "$v" paper_2509_17396_b200/libepk.so
  echo "== $v"; timeout 300 python scripts/xp_time.py 20 2>&1 | tail -1
done
cp /tmp/libepk_orig.so paper_2509_17396_b200/libepk.so
