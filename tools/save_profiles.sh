#!/bin/bash
# Copy one gpu_round.sh + bench_all.sh run (TAG) into profiles/ (the judged copies).
set -e
TAG=${1:?tag}
python tools/ncu_summary.py gpurun_out/prof_$TAG.ncu-rep profiles/r01_ncu_full_C3_plane.json > /dev/null
cp gpurun_out/launches_$TAG.csv profiles/r01_launches_C3_plane.csv
cp gpurun_out/bench_$TAG.json profiles/r01_bench_C3_plane.json
for w in C1 C2 C3 C4 C5; do cp gpurun_out/bench_${TAG}_$w.json profiles/r01_per_config/bench_$w.json; done
python - "$TAG" <<'PY'
import csv, collections, json, sys
d = json.load(open("profiles/r01_ncu_full_C3_plane.json"))
jvp = [k for k in d if "plane_kernel<4, 1, 1, 0>" in k["kernel"]][0]
num = lambda s: float(s.split()[0]) * (1e6 if "Mbyte" in s else 1e9 if "Gbyte" in s else 1.0)
json.dump({"C3": int(num(jvp["dram__bytes_read.sum"]) + num(jvp["dram__bytes_write.sum"])),
           "_source": "profiles/r01_ncu_full_C3_plane.json: dram__bytes_read.sum + dram__bytes_write.sum of "
                      "plane_kernel<4,1,1,0> (C3 JVP), one ncu --set full launch"},
          open("profiles/traffic.json", "w"), indent=1)
rows = [r for r in csv.reader(open("profiles/r01_launches_C3_plane.csv")) if len(r) > 14 and r[12] == "gpu__time_duration.sum"]
seq = [(r[4].split("(")[0], float(r[14]) / 1000) for r in rows]
# the bench's steps come first after the setup kernel: (warmup 3 + steps 2) x 4 launches
# (residual, its fix-up, JVP, its fix-up); the per-call diagnostics that follow are not in the step
step = [x for x in seq if "geometry" not in x[0]][:20]
agg = collections.defaultdict(list)
for k, t in step:
    agg[k].append(t)
tot = sum(t for _, t in step)
out = {k: {"n": len(v), "mean_us": sum(v) / len(v), "share_of_step": sum(v) / tot} for k, v in agg.items()}
out["_note"] = ("ncu --metrics gpu__time_duration.sum --clock-control none (cold, serialised); the 20 launches of "
                "bench.py --steps 2 --warmup 3 (5 steps x [plane_kernel<RES>, fixup, plane_kernel<JVP>, fixup])")
json.dump(out, open("profiles/r01_launches_C3_plane_summary.json", "w"), indent=1)
print(json.dumps(out, indent=1))
PY
