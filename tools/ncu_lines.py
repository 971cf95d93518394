#!/usr/bin/env python
"""Per-CUDA-line stall attribution from an ncu report (--page source sass,cuda).
usage: ncu_lines.py report.ncu-rep kernel_substring [stall_column] [top]"""
import collections
import csv
import io
import subprocess
import sys

rep, ksub = sys.argv[1], sys.argv[2]
col = sys.argv[3] if len(sys.argv) > 3 else "Warp Stall Sampling (All Samples)"
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
func = fname = hdr = None
agg = collections.defaultdict(lambda: [0, 0, ""])
tot = 0
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        func = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if func is None or ksub not in func or hdr is None:
        continue
    try:
        w = int(r[hdr.index(col)] or 0)
        n = int(r[hdr.index("Instructions Executed")] or 0)
    except (ValueError, IndexError):
        continue
    key = (fname, r[0])
    agg[key][0] += w
    agg[key][1] += n
    agg[key][2] = r[1][:95]
    tot += w
for (f, l), (w, n, src) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{f}:{l:5s} {100 * w / max(tot, 1):5.1f}%  inst {n:10d}  {src}")
