"""Quick per-call timer (CUDA events, same stream): python tools/kt.py C5 jvp residual design ...
Not a bench line; for iteration on the GPU box."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_00746_b200 as fe  # noqa: E402
import workloads as W  # noqa: E402


def main():
    wname = sys.argv[1]
    calls = sys.argv[2:] or ["residual", "jvp"]
    reps = int(os.environ.get("REPS", "50"))
    w = W.CONFIGS[wname]
    if os.environ.get("N"):
        w = w.resized(int(os.environ["N"]))
    d = W.draw(w)
    rho = torch.as_tensor(d["rho"]).cuda() if "rho" in d else None
    op = fe.from_workload(w, verts=d["verts"], rho=rho)
    u = torch.as_tensor(d["u"]).cuda()
    v = torch.as_tensor(d.get("v", d.get("lam"))).cuda()
    lam = torch.as_tensor(d.get("lam", d.get("v"))).cuda()
    out = torch.empty_like(u)
    out2 = torch.empty_like(u)
    g = torch.empty(w.n_elems, dtype=torch.float64, device="cuda")
    nn = (w.k + 1) ** 3
    nem = min(16384 if w.k <= 3 else 512, w.n_elems)   # Q4..Q6: K_e up to 941 KB per element
    Ke = torch.empty((nem, nn, nn), dtype=torch.float64, device="cuda")
    fns = {
        "residual": lambda: op.residual(u, out=out),
        "jvp": lambda: op.jvp(u, v, out=out),
        "jvp_res": lambda: op.jvp_res(u, v, out=(out2, out)),
        "vjp": lambda: op.vjp(u, v, out=out),
        "design": lambda: op.design_grad(u, lam, out=g),
        "res_design": lambda: op.res_design_grad(u, lam, out=(out, g)),
        "linearize": lambda: op.linearize(u, out=out),
        "jvp_lin": lambda: op.jvp_lin(v, out=out),
        "jacobi_diag": lambda: op.jacobi_diag(out=out),
        "elemat": lambda: op.element_matrices(u, 0, nem, out=Ke),
        "elm": lambda: op.element_matrices(u, 0, nem, elm=True, out=Ke),
    }
    for c in calls:
        if c in ("jvp_lin", "jacobi_diag"):
            op.linearize(u, out=out2)
        f = fns[c]
        for _ in range(5):
            f()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            f()
            b.record()
            ts.append((a, b))
        torch.cuda.synchronize()
        t = [x.elapsed_time(y) * 1e3 for x, y in ts]
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            f()
        b.record()
        torch.cuda.synchronize()
        print(f"{wname} {c:10s} per-call mean {statistics.mean(t):8.1f} med {statistics.median(t):8.1f} "
              f"min {min(t):8.1f} us | back-to-back {a.elapsed_time(b) * 1e3 / reps:8.1f} us", flush=True)


if __name__ == "__main__":
    main()
