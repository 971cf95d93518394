#!/bin/bash
# One ncu --set full capture per (workload, call, kernel regex), after the same command
# ran clean without ncu; keeps the counter summary, per-opcode (SASS) and per-line stall
# tables under gpurun_out/prof/. Usage: tools/gpu_prof.sh TAG WORKLOAD CALL KREGEX [SKIP]
set -u
TAG=$1; W=$2; C=$3; K=$4; SKIP=${5:-2}
O=gpurun_out/prof
mkdir -p $O
REPS=3 python tools/kt.py $W $C > $O/kt_$TAG.txt 2>&1 || { echo "kt $TAG failed"; cat $O/kt_$TAG.txt; exit 1; }
cat $O/kt_$TAG.txt
REPS=2 ncu --set full --clock-control none --import-source on -k regex:"$K" -s $SKIP -c 1 \
   -o $O/$TAG python tools/kt.py $W $C > $O/ncu_$TAG.log 2>&1
echo "ncu $TAG rc=$?"
python tools/ncu_summary.py $O/$TAG.ncu-rep $O/$TAG.json > /dev/null 2>&1
ncu -i $O/$TAG.ncu-rep --page source --csv --print-source cuda,sass > /tmp/src_$TAG.csv 2>/dev/null
ncu -i $O/$TAG.ncu-rep --page source --csv --print-source sass > /tmp/sass_$TAG.csv 2>/dev/null
python tools/line_hot.py /tmp/src_$TAG.csv 40 > $O/${TAG}_lines.txt 2>&1
python tools/sass_hot.py /tmp/sass_$TAG.csv > $O/${TAG}_ops.txt 2>&1
rm -f $O/$TAG.ncu-rep
