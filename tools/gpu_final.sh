#!/bin/bash
# Round-2 closing evidence (one gpurun call): GPU tests, smoke(), the default bench line,
# per-config bench lines, the ncu launch list of the default bench command, and ncu
# --set full captures of the Q6 tensor-core kernels after the last changes.
set -u
O=${O:-gpurun_out/r02f}
mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
python bench.py > $O/bench_C3.json 2> $O/bench_C3.err; echo "bench rc=$?"
for w in C5 C2 C4 C1; do
  timeout 900 python bench.py --workload $w --steps 200 --warmup 5 > $O/bench_$w.json 2> $O/bench_$w.err
  echo "bench $w rc=$?"
done
CMD="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > $O/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C3.csv $CMD > $O/ncu_launch.log 2>&1
echo "ncu launches rc=$?"
CMD4="python bench.py --workload C4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD4 > $O/plain4.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv -c 200 --log-file $O/launches_C4.csv $CMD4 > $O/ncu_launch4.log 2>&1
echo "ncu launches C4 rc=$?"
mkdir -p gpurun_out/prof
bash tools/gpu_prof.sh c4final_jvp C4 jvp q6tc_perl
bash tools/gpu_prof.sh c4final_res C4 residual q6tc_perl
bash tools/gpu_prof.sh c4final_asm C4 jvp evec_assemble
bash tools/gpu_prof.sh c4final_emhi C4 elemat elemat_hi 1
bash tools/gpu_prof.sh c4final_jvplin C4 jvp_lin q6tc_perl
bash tools/gpu_prof.sh c4final_diag C4 jacobi_diag q6tc_diag 1
python tools/newton_time.py 5 > $O/newton_time.txt 2>&1
cp gpurun_out/prof/c4final_* $O/ 2>/dev/null
python tools/link_bw.py > $O/link_bw.json 2>&1
