#!/bin/bash
# One GPU call: parity tests, the default bench line, the ncu launch list and one
# --set full capture of the fused kernels (each ncu only after its command exited 0).
set -u
mkdir -p gpurun_out
TAG=${TAG:-r01}
python -m pytest ${TESTS:-tests} -x -q -m gpu > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu_$TAG.log
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
cat gpurun_out/bench_$TAG.json; tail -3 gpurun_out/bench_$TAG.err
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
if [ "${NCU:-1}" = "1" ]; then
  $CMD > gpurun_out/plain_$TAG.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1
  echo "ncu launches rc=$?"
  $CMD > gpurun_out/plain2_$TAG.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"plane_kernel|fixup" -s 12 -c 4 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
  echo "ncu full rc=$?"
fi
