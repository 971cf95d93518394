#!/bin/bash
# A/B the abtest/libfeod_<v>.so variants (VARIANTS) on WL workloads via exp_variants.py.
for v in ${VARIANTS:-base}; do
  cp abtest/libfeod_$v.so paper_2506_00746_b200/libfeod.so
  echo "== $v"; ONLY=${ONLY:-} timeout 200 python tools/exp_variants.py ${WL:-C3 C2} | grep label
done
