#!/bin/bash
# ncu --set full of the kernels beyond the bench step (C3): J^T w, linearize, J v from the
# stored linearisation, the element-tangent DMMA kernel, the Jacobi diagonal.
mkdir -p gpurun_out
TAG=${TAG:-dev}
CMD="python bench.py --workload C3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plainx_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on \
  -k regex:"plane_kernel<4, (4|5|6)|elemat_kernel<4, 1, 0, 0>|diag_color" -c 5 -o gpurun_out/profx_$TAG $CMD > gpurun_out/ncux_$TAG.log 2>&1
echo "ncu extra rc=$?"
