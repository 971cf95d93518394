#!/usr/bin/env python
"""Aggregate an ncu `--page source --print-source cuda,sass --csv` export by CUDA
source line: stall samples, executed warp-instructions, top stall reasons."""
import collections
import csv
import io
import sys

txt = open(sys.argv[1]).read()
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
blocks = txt.split('"File Path"')
agg = collections.defaultdict(collections.Counter)
srcline = {}
total = 0
for b in blocks[1:]:
    lines = b.splitlines()
    fpath = lines[0].strip(',"')
    fname = fpath.split("/")[-1]
    rows = list(csv.reader(io.StringIO("\n".join(lines[2:]))))
    h = rows[0]
    iS = h.index("Warp Stall Sampling (All Samples)")
    iE = h.index("Instructions Executed")
    stall_cols = [(i, k) for i, k in enumerate(h) if k.startswith("stall_") and "Not Issued" not in k]
    cur = None
    for r in rows[1:]:
        if not r:
            continue
        if r[0].strip():
            cur = (fname, int(r[0]))
            srcline[cur] = r[1].strip()[:70]
        if len(r) <= iS or not r[2].strip() or cur is None:
            continue
        try:
            s = float(r[iS] or 0)
            e = float(r[iE] or 0)
        except ValueError:
            continue
        agg[cur]["samples"] += s
        agg[cur]["inst"] += e
        total += s
        for i, k in stall_cols:
            try:
                agg[cur][k] += float(r[i] or 0)
            except ValueError:
                pass
print(f"total samples {total:.0f}")
for key, v in sorted(agg.items(), key=lambda x: -x[1]["samples"])[:top]:
    st = sorted(((k[6:], v[k]) for k in v if k.startswith("stall_")), key=lambda x: -x[1])[:3]
    sts = " ".join(f"{k}:{int(c)}" for k, c in st)
    print(f"{key[0]}:{key[1]:<4d} {100 * v['samples'] / total:5.1f}% inst {v['inst'] / 1e6:6.2f}M  {sts:45s} | {srcline.get(key, '')}")
