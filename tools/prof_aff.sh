#!/bin/bash
# ncu --set full of the C3-sized affine ("flip") JVP kernel via tools/exp_variants.py
TAG=${TAG:-dev}; WLD=${WLD:-C3}; SKIP=${SKIP:-3}
ONLY=flip REPS=2 python tools/exp_variants.py $WLD > gpurun_out/plain_$TAG.log 2>&1 && \
ONLY=flip REPS=2 ncu --set full --clock-control none --import-source on -k regex:plane_kernel -s $SKIP -c 1 -o gpurun_out/prof_$TAG python tools/exp_variants.py $WLD > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc=$?"
