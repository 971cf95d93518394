#!/bin/bash
# Quick GPU iteration: parity tests, then per-config bench lines (no ncu).
mkdir -p gpurun_out
TAG=${TAG:-dev}
timeout 600 python -m pytest ${TESTS:-tests} -x -q -m gpu > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_$TAG.log
for w in ${WL:-C3 C2 C5 C4 C1}; do
  timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_$w.json 2> gpurun_out/bench_${TAG}_$w.err
  echo "$w rc=$?"; tail -2 gpurun_out/bench_${TAG}_$w.err
done
python - <<'PY'
import json, os
tag = os.environ.get("TAG", "dev")
for w in os.environ.get("WL", "C3 C2 C5 C4 C1").split():
    try:
        d = json.load(open(f"gpurun_out/bench_{tag}_{w}.json"))
    except Exception as e:
        print(w, "failed", e); continue
    c = d["calls"]
    print(f"{w}: res {c['residual']['us']:.1f} us (hbm {c['residual']['hbm_frac']:.2f}, fp64 {c['residual']['fp64_frac']:.2f}) | "
          f"jvp {c['jvp']['us']:.1f} us kernel {c['jvp']['fused_kernel_us']:.1f} (hbm {c['jvp']['hbm_frac']:.2f}, fp64 {c['jvp']['fp64_frac']:.2f}) | frac {d['roofline']['frac']:.3f}")
PY
