#!/usr/bin/env python
"""Diagnostics: per-CTA start/end times of the persistent plane kernel (library
built with -DFEOD_PROFILE_TAIL), to size the tail where CTAs have run out of
bricks. Not a bench line."""
import collections
import os
import subprocess
import sys

if len(sys.argv) > 1 and sys.argv[1] == "child":
    import torch
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_2506_00746_b200 as fe
    import workloads as W
    w = getattr(W, sys.argv[2])
    d = W.draw(w)
    op = fe.from_workload(w, verts=d["verts"])
    u, v = torch.as_tensor(d["u"]).cuda(), torch.as_tensor(d["v"]).cuda()
    for _ in range(3):
        op.jvp(u, v)
        op.residual(u)
    torch.cuda.synchronize()
    sys.exit(0)

wl = sys.argv[1] if len(sys.argv) > 1 else "C3"
out = subprocess.run([sys.executable, __file__, "child", wl], capture_output=True, text=True).stdout
calls = collections.defaultdict(list)
for line in out.splitlines():
    if line.startswith("TAIL"):
        _, mode, base, blk, L, t0, t1 = line.split()
        calls[(int(mode), int(base))].append((int(blk), int(L), int(t0), int(t1)))
for (mode, base), rows in sorted(calls.items(), key=lambda kv: kv[0][1])[-2:]:
    t0 = min(r[2] for r in rows)
    ends = sorted((r[3] - t0) / 1e3 for r in rows)
    starts = sorted((r[2] - t0) / 1e3 for r in rows)
    span = ends[-1]
    busy = sum(e - s for e, s in zip(sorted(r[3] for r in rows), sorted(r[2] for r in rows))) / 1e3
    layers = collections.Counter(r[1] for r in rows)
    print(f"mode {mode}: {len(rows)} CTAs, span {span:.1f} us, starts last {starts[-1]:.1f} us, "
          f"ends min {ends[0]:.1f} p10 {ends[len(ends)//10]:.1f} p50 {ends[len(ends)//2]:.1f} p90 {ends[9*len(ends)//10]:.1f}, "
          f"busy fraction {busy / (span * len(rows)):.3f}; layers per CTA {sorted(layers.items())}")
