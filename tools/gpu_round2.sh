#!/bin/bash
# Round-2 evidence run (one gpurun call): GPU tests, the default bench line, per-config
# bench lines, the ncu launch list of the default bench command, and ncu --set full
# captures of the JVP / residual kernels of C2, C3, C4, C5 (each ncu only after the
# same command exited 0 without ncu). Output: gpurun_out/r02/.
set -u
O=gpurun_out/r02
mkdir -p $O
if [ "${TESTS:-1}" = "1" ]; then
  timeout 1500 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
fi
python bench.py > $O/bench_C3.json 2> $O/bench_C3.err; echo "bench rc=$?"; tail -2 $O/bench_C3.err
for w in C5 C2 C4 C1; do
  timeout 600 python bench.py --workload $w --steps 200 --warmup 5 > $O/bench_$w.json 2> $O/bench_$w.err
  echo "bench $w rc=$?"; tail -1 $O/bench_$w.err
done
CMD="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > $O/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C3.csv $CMD > $O/ncu_launch.log 2>&1
echo "ncu launches rc=$?"
for w in C2 C3 C4 C5; do
  REPS=2 python tools/kt.py $w jvp residual > /dev/null 2>&1 && \
  REPS=2 ncu --set full --clock-control none --import-source on -k regex:"col_kernel|plane_kernel|fixup_kernel" -s 6 -c 3 \
     -o $O/full_$w python tools/kt.py $w jvp residual > $O/ncu_full_$w.log 2>&1
  echo "ncu full $w rc=$?"
  # keep the summaries (gpurun brings back <= 64 MiB): counters, per-line and per-region stalls
  python tools/ncu_summary.py $O/full_$w.ncu-rep > $O/full_$w.json 2>&1
  ncu -i $O/full_$w.ncu-rep --page source --csv --print-source cuda,sass > /tmp/src_$w.csv 2>/dev/null
  python tools/line_hot.py /tmp/src_$w.csv 40 > $O/full_${w}_lines.txt 2>&1
  python tools/region_hot.py /tmp/src_$w.csv > $O/full_${w}_regions.txt 2>&1
  rm -f $O/full_$w.ncu-rep
done
