#!/usr/bin/env python
"""Per-opcode aggregation of an ncu source-page CSV (SASS view): stall samples,
executed instructions, shared-memory wavefronts. Usage: sass_hot.py src.csv [kernel-substring]"""
import collections
import csv
import io
import sys

txt = open(sys.argv[1]).read()
want = sys.argv[2] if len(sys.argv) > 2 else ""
for b in txt.split('"Kernel Name"')[1:]:
    lines = b.splitlines()
    name = lines[0]
    if want not in name:
        continue
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    h = rows[0]
    ix = {k: h.index(k) for k in ["Source", "Warp Stall Sampling (All Samples)", "Instructions Executed",
                                 "L1 Wavefronts Shared", "L1 Wavefronts Shared Ideal", "stall_wait", "stall_barrier",
                                 "stall_long_sb", "stall_short_sb", "stall_mio", "stall_math"] if k in h}
    agg = collections.defaultdict(lambda: collections.Counter())
    for r in rows[1:]:
        if len(r) < len(h):
            continue
        s = r[ix["Source"]].strip()
        if not s:
            continue
        tok = s.split()
        op = tok[1] if tok[0].startswith("@") else tok[0]
        base = op.split(".")[0]
        if base in ("LDS", "STS", "LDG", "STG", "SHFL", "LDGSTS"):
            base = op
        for k in ix:
            if k == "Source":
                continue
            try:
                agg[base][k] += float(r[ix[k]] or 0) if k in ix else 0.0
            except ValueError:
                pass
    tot = sum(v["Warp Stall Sampling (All Samples)"] for v in agg.values())
    toti = sum(v["Instructions Executed"] for v in agg.values())
    print(name[:100])
    print(f"{'op':22s} {'samp%':>6s} {'inst%':>6s} {'inst(M)':>8s} {'wf(M)':>7s} {'wfideal':>7s} wait barr lsb ssb mio math")
    for op, v in sorted(agg.items(), key=lambda x: -x[1]["Warp Stall Sampling (All Samples)"])[:28]:
        s = v["Warp Stall Sampling (All Samples)"]
        print(f"{op:22s} {100*s/tot:6.1f} {100*v['Instructions Executed']/toti:6.1f} {v['Instructions Executed']/1e6:8.2f} "
              f"{v['L1 Wavefronts Shared']/1e6:7.2f} {v['L1 Wavefronts Shared Ideal']/1e6:7.2f} "
              f"{int(v['stall_wait'])} {int(v['stall_barrier'])} {int(v['stall_long_sb'])} {int(v['stall_short_sb'])} {int(v['stall_mio'])} {int(v['stall_math'])}")
