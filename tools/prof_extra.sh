#!/bin/bash
# ncu --set full, one launch each, of the kernels beyond the bench step (C3): J^T w (mode 4),
# linearize (5), J v from the stored linearisation (6), the element-tangent DMMA kernel (RES).
mkdir -p gpurun_out
TAG=${TAG:-dev}
CMD="python bench.py --workload C3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plainx_$TAG.log 2>&1 || { echo "plain run failed"; exit 1; }
i=0
for rx in 'plane_kernel<\(int\)4, \(int\)4' 'plane_kernel<\(int\)4, \(int\)5' 'plane_kernel<\(int\)4, \(int\)6' \
          'elemat_kernel<\(int\)4, \(int\)1, \(bool\)0, \(bool\)0>'; do
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$rx" -c 1 \
    -o gpurun_out/profx_${TAG}_$i $CMD > gpurun_out/ncux_${TAG}_$i.log 2>&1
  echo "ncu $i rc=$?"
  i=$((i+1))
done
