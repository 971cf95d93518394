#!/bin/bash
# Step 0: sustained FP64 + HBM probe with clocks sampled during the run.
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/peaks_clocks.csv &
SMI=$!
./tools/fp64_peak > gpurun_out/peaks_fp64.json
kill $SMI
cat gpurun_out/peaks_fp64.json
nproc; grep -m1 "model name" /proc/cpuinfo; python -c "import os; print(len(os.sched_getaffinity(0)))"
