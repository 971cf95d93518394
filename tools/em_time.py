#!/usr/bin/env python
"""Diagnostics: ns/element of feod_element_matrices (RES and ELM) at Q4..Q6 for the
library named by FEOD_LIB (experiment builds). Not a bench line."""
import dataclasses
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_00746_b200 as fe  # noqa: E402
import workloads as W  # noqa: E402


def t_call(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


out = {"lib": os.environ.get("FEOD_LIB", "default")}
cases = [("Q4", dataclasses.replace(W.C3, k=4, q=5).resized(24)), ("Q5", dataclasses.replace(W.C2, k=5, q=6).resized(20)),
         ("Q6", W.C4)]
for name, w in cases:
    d = W.draw(w)
    rho = torch.as_tensor(d["rho"]).cuda() if "rho" in d else None
    op = fe.from_workload(w, verts=d["verts"], rho=rho)
    u = torch.as_tensor(d["u"]).cuda()
    nn = (w.k + 1) ** 3
    ne = min(op.n_elems, 1024)
    Ke = torch.empty((ne, nn, nn), dtype=torch.float64, device="cuda")
    for elm in (False,) if os.environ.get("RES_ONLY") else (False, True):
        us = t_call(lambda: op.element_matrices(u, 0, ne, elm=elm, out=Ke))
        tf = 2.0 * nn * nn * 3 * w.q ** 3 * ne / (us * 1e-6) / 1e12
        out[f"{name}_{'ELM' if elm else 'RES'}_ns_per_el"] = us * 1e3 / ne
        if not elm:
            out[f"{name}_RES_gemm_tflops"] = tf
print(json.dumps(out))
