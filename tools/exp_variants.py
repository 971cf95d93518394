#!/usr/bin/env python
"""Diagnostics: time residual / JVP kernels of C3-sized variants (perturbed vs
affine mesh, model) to separate the metric stream from the compute, plus a plain
read-bandwidth reference of the same byte count. Not a bench line."""
import dataclasses
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_00746_b200 as fe  # noqa: E402
import workloads as W  # noqa: E402


REPS = int(os.environ.get("REPS", "20"))


def t_call(fn, reps=None):
    reps = reps or REPS
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


def run(w, label):
    d = W.draw(w)
    rho = torch.as_tensor(d["rho"]).cuda() if "rho" in d else None
    op = fe.from_workload(w, verts=d["verts"], rho=rho)
    u, v = torch.as_tensor(d["u"]).cuda(), torch.as_tensor(d["v"]).cuda()
    r, Jv = torch.empty_like(u), torch.empty_like(u)
    res = t_call(lambda: op.residual(u, out=r))
    jvp = t_call(lambda: op.jvp(u, v, out=Jv))
    ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    ev[0].record()
    ev[1].record()
    torch.cuda.synchronize()
    op.profile_next(*ev)
    op.jvp(u, v, out=Jv)
    torch.cuda.synchronize()
    kern = ev[0].elapsed_time(ev[1]) * 1e3
    out = {"label": label, "res_us": res, "jvp_us": jvp, "jvp_kernel_us": kern}
    print(json.dumps(out), flush=True)
    del op


def main():
    torch.cuda.set_device(0)
    names = sys.argv[1:] or ["C3"]
    only = os.environ.get("ONLY")   # "flip": only the flipped-mesh variant
    for nm in names:
        w = W.CONFIGS[nm]
        if only != "flip":
            run(w, nm)
        run(dataclasses.replace(w, perturbed=not w.perturbed, name=nm + "-flipmesh"), nm + " mesh flipped")
    if only:
        return
    # read-bandwidth reference: sum of an 805 MB fp64 buffer
    x = torch.empty(805_306_368 // 8, dtype=torch.float64, device="cuda").uniform_()
    us = t_call(lambda: x.sum())
    print(json.dumps({"label": "torch sum 805MB", "us": us, "GBps": 805.3e6 / us / 1e3}))


if __name__ == "__main__":
    main()
