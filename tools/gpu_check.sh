#!/bin/bash
# Mid-round check (one gpurun call): full GPU suite, smoke(), the driver's bench command.
set -u
O=gpurun_out/${TAG:-chk}
mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench_C3.json 2> $O/bench_C3.err; echo "bench rc=$?"; tail -2 $O/bench_C3.err
python -c "
import json; d=json.load(open('$O/bench_C3.json')); print(d['value'], d['roofline']['frac'], d['e2e']['value'], d['clocks'])"
