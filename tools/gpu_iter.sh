#!/bin/bash
# Iteration run: GPU tests (optional subset), then quick per-call timings.
# Usage: TESTS="tests -m gpu" KT="C4:jvp,residual C1:jvp" tools/gpu_iter.sh
set -u
O=gpurun_out/iter
mkdir -p $O
if [ -n "${TESTS:-}" ]; then
  timeout 1200 python -m pytest ${TESTS} -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
fi
for spec in ${KT:-}; do
  w=${spec%%:*}; calls=${spec#*:}
  timeout 300 env ${KTENV:-} python tools/kt.py $w ${calls//,/ } 2>&1 | tee -a $O/kt.log
done
