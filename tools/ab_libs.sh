#!/bin/bash
# A/B the abtest/libfeod_<v>.so variants (VARIANTS, "base" = the in-tree build) on the
# WL workloads and CALLS (tools/kt.py); the in-tree library is never overwritten.
for v in ${VARIANTS:-base}; do
  lib=abtest/libfeod_$v.so; [ "$v" = base ] && lib=paper_2506_00746_b200/libfeod.so
  for w in ${WL:-C5}; do echo "== $v"; FEOD_LIB=$PWD/$lib timeout 300 python tools/kt.py $w ${CALLS:-jvp residual}; done
done
