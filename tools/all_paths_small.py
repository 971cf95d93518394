#!/usr/bin/env python
"""Every entry point on small cases (ragged bricks, two z-slabs): a quick all-paths run,
e.g. under a memory checker where one is available (compute-sanitizer is closed on the
GPU pool this repo is measured on). Not a test; parity is in tests/."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_00746_b200 as fe  # noqa: E402
import workloads as W  # noqa: E402

for w, n in ((W.C1, 4), (W.C2, 11), (W.C3, 5), (W.C3, 18), (W.C4, 3), (W.C5, 9)):
    ww = w.resized(n)
    d = W.draw(ww)
    rho = torch.as_tensor(d["rho"]).cuda() if "rho" in d else None
    op = fe.from_workload(ww, verts=d["verts"], rho=rho)
    u, v = torch.as_tensor(d["u"]).cuda(), torch.as_tensor(d["v"]).cuda()
    op.residual(u); op.jvp(u, v); op.jvp_res(u, v); op.vjp(u, v)
    op.linearize(u); op.jvp_lin(v); op.jacobi_diag()
    if ww.k <= 3:
        op.element_matrices(u, 0, min(8, op.n_elems))
    if "rho" in d:
        op.design_grad(u, v)
        op.adjoint_solve(u, v, iters=3)
    torch.cuda.synchronize()
    print(ww.name, "ok", flush=True)
