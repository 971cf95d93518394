"""Time feod_newton_cg (A15: 5 x 20 from u0 = 0) at C4 for the three Jacobian variants, with
and without the fused CG update: python tools/newton_time.py [reps]. Not a bench line."""
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_00746_b200 as fe  # noqa: E402
import workloads as W  # noqa: E402

w = W.C4
d = W.draw(w)
op = fe.from_workload(w, verts=d["verts"])
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
for fusion in (0, 1):
    op.set_cg_fusion(fusion)
    for stored in (0, 1, 2):
        op.set_newton_linearization(stored)
        u0 = torch.zeros(w.n_dofs, dtype=torch.float64, device="cuda")
        op.newton_cg(u0.clone(), 5, 20)
        ts = []
        for _ in range(reps):
            u = u0.clone()
            torch.cuda.synchronize()
            t = time.perf_counter()
            _, norms = op.newton_cg(u, 5, 20)
            torch.cuda.synchronize()
            ts.append((time.perf_counter() - t) * 1e3)
        print(f"fusion={fusion} stored={stored}: median {statistics.median(ts):.2f} ms min {min(ts):.2f} ms "
              f"norms[-1]={norms[-1]:.6e}", flush=True)
