#!/bin/bash
# Per-config numbers (diagnostics; the bench line of record is bench.py's default C3 workload).
mkdir -p gpurun_out
TAG=${TAG:-r01}
for w in C1 C2 C3 C4 C5; do
  python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_$w.json 2> gpurun_out/bench_${TAG}_$w.err
  echo "$w rc=$?"
done
python - <<'PY'
import json, glob, os
tag = os.environ.get("TAG", "r01")
for w in ["C1","C2","C3","C4","C5"]:
    try:
        d = json.load(open(f"gpurun_out/bench_{tag}_{w}.json"))
    except Exception as e:
        print(w, "failed", e); continue
    c = d["calls"]
    print(f"{w}: res {c['residual']['us']:.1f} us ({c['residual']['gdof_s']:.1f} GDOF/s, hbm {c['residual']['hbm_frac']:.2f}, fp64 {c['residual']['fp64_frac']:.2f}) | "
          f"jvp {c['jvp']['us']:.1f} us ({c['jvp']['gdof_s']:.1f} GDOF/s, hbm {c['jvp']['hbm_frac']:.2f}, fp64 {c['jvp']['fp64_frac']:.2f}) | roofline frac {d['roofline']['frac']:.3f}")
PY
