#!/bin/bash
# One ncu --set full capture of the fused residual + JVP kernels of a workload (after a clean run).
mkdir -p gpurun_out
TAG=${TAG:-dev}; WLD=${WLD:-C3}
CMD="python bench.py --workload $WLD --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:plane_kernel -s 6 -c 2 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "ncu rc=$?"
