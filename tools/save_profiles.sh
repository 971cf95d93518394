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
agg = collections.defaultdict(list)
for r in rows:
    agg[r[4].split("(")[0]].append(float(r[14]) / 1000)
tot = sum(sum(v) for k, v in agg.items() if "geometry" not in k)
out = {k: {"n": len(v), "mean_us": sum(v) / len(v), "share_of_step": (sum(v) / tot if "geometry" not in k else None)}
       for k, v in agg.items()}
json.dump(out, open("profiles/r01_launches_C3_plane_summary.json", "w"), indent=1)
print(json.dumps(out, indent=1))
PY
