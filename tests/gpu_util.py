"""Helpers shared by the GPU parity tests (marshalling only, no method arithmetic)."""
import numpy as np

import oracle as O
import workloads as W


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def problem(w, d):
    return O.Problem.from_workload(w, verts=d["verts"], rho=d.get("rho"))


def operator(w, d):
    import torch
    import paper_2506_00746_b200 as fe
    rho = torch.as_tensor(d["rho"]).cuda() if "rho" in d else None
    return fe.from_workload(w, verts=d["verts"], rho=rho)


def cuda(x):
    import torch
    return torch.as_tensor(np.asarray(x, dtype=np.float64)).cuda()


def host(t):
    return t.detach().cpu().numpy()
