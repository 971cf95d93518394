set -e
for v in minb3 minb4; do
  cp abtest/libfeod_$v.so paper_2506_00746_b200/libfeod.so
  echo "== $v"; timeout 120 python tools/exp_variants.py C3 C2 | grep label
done
