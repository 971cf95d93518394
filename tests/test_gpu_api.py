"""GPU parity at the API edge and binding checks.

* general-exponent p-Laplacian (the pow branch of dual.cuh / physics.cuh, not the
  p = 2, 3, 4 shortcuts) on perturbed meshes for both kernel families;
* reading A20: eps = 0 with exactly zero gradients (the defined limit, no NaN);
* out= / device / length validation in the binding, one handle driven on two streams.
"""
import dataclasses

import numpy as np
import pytest

import oracle as O
import workloads as W
from gpu_util import rel_l2, problem, operator, cuda, host

pytestmark = pytest.mark.gpu
TOL = 1e-11

GENP = [(dataclasses.replace(W.C2, k=1, q=2), 7, 2.5), (dataclasses.replace(W.C2, k=2, q=3), 5, 3.5),
        (dataclasses.replace(W.C3, model=W.PLAPLACE, eps=1e-2, u_scale=1.0), 5, 2.5),
        (dataclasses.replace(W.C4, perturbed=True), 2, 3.5)]


@pytest.mark.parametrize("w,n,p", GENP, ids=[f"Q{w.k}n{n}p{p}" for w, n, p in GENP])
def test_general_exponent_parity(w, n, p):
    ww = dataclasses.replace(w.resized(n), p=p, eps=w.eps or 1e-2)
    d = W.draw(ww)
    pr, op = problem(ww, d), operator(ww, d)
    assert rel_l2(host(op.residual(cuda(d["u"]))), O.residual(pr, d["u"])) <= TOL
    assert rel_l2(host(op.jvp(cuda(d["u"]), cuda(d["v"]))), O.jvp(pr, d["u"], d["v"])) <= TOL
    assert rel_l2(host(op.vjp(cuda(d["u"]), cuda(d["v"]))), O.vjp(pr, d["u"], d["v"])) <= TOL


A20 = [(2, 4, 2.5), (2, 4, 3.0), (1, 6, 3.5), (3, 3, 4.0), (3, 3, 2.5)]


@pytest.mark.parametrize("k,n,p", A20, ids=[f"Q{k}n{n}p{p}" for k, n, p in A20])
def test_a20_eps0_zero_gradient_parity(k, n, p):
    """eps = 0, u random on a corner box of nodes and 0 elsewhere: grad u = 0 exactly on
    every element away from the box (both sides contract zeros), generic elsewhere (a
    gradient that is zero only up to rounding would make dD/dg ~ |g|^(p-2) noise)."""
    w = dataclasses.replace(W.C1, n=n, k=k, q=k + 1, p=p, eps=0.0, name=f"A20Q{k}")
    d = W.draw(w)
    m = k * n + 1
    I = np.arange(w.n_dofs)
    box = (I % m <= k + 1) & ((I // m) % m <= k + 1) & (I // (m * m) <= k + 1)
    u = np.where(box, d["u"], 0.0)
    pr, op = problem(w, d), operator(w, d)
    r = host(op.residual(cuda(u)))
    Jv = host(op.jvp(cuda(u), cuda(d["v"])))
    JTw = host(op.vjp(cuda(u), cuda(d["v"])))
    assert np.all(np.isfinite(r)) and np.all(np.isfinite(Jv)) and np.all(np.isfinite(JTw))
    assert rel_l2(r, O.residual(pr, u)) <= TOL
    assert rel_l2(Jv, O.jvp(pr, u, d["v"])) <= TOL
    assert rel_l2(JTw, O.vjp(pr, u, d["v"])) <= TOL


def _small():
    w = W.C5.resized(6)
    d = W.draw(w)
    return w, d, operator(w, d)


def test_out_validation():
    import torch
    import paper_2506_00746_b200 as fe
    w, d, op = _small()
    u, v = cuda(d["u"]), cuda(d["v"])
    for bad in (torch.empty(w.n_dofs - 1, dtype=torch.float64, device="cuda"),
                torch.empty(w.n_dofs, dtype=torch.float32, device="cuda"),
                torch.empty(2 * w.n_dofs, dtype=torch.float64, device="cuda")[::2],
                torch.empty(w.n_dofs, dtype=torch.float64)):
        with pytest.raises(fe.FeodError):
            op.jvp(u, v, out=bad)
        with pytest.raises(fe.FeodError):
            op.residual(u, out=bad)
    with pytest.raises(fe.FeodError):
        op.design_grad(u, v, out=torch.empty(w.n_elems - 1, dtype=torch.float64, device="cuda"))
    with pytest.raises(fe.FeodError):
        op.dot(u, torch.zeros(w.n_dofs - 3, dtype=torch.float64, device="cuda"))
    with pytest.raises(fe.FeodError):
        op.apply_host(1, d["u"], d["v"], out=torch.empty(w.n_dofs - 1, dtype=torch.float64))
    good = torch.empty(w.n_dofs, dtype=torch.float64, device="cuda")
    assert op.jvp(u, v, out=good) is good


def test_one_handle_two_streams_bitwise():
    """feod_set_stream orders the old stream's work before the new stream's: alternating
    streams on one handle (shared tickets / shell / epochs) gives the same bits."""
    import torch
    w, d, op = _small()
    u, v = cuda(d["u"]), cuda(d["v"])
    ref = op.jvp(u, v).clone()
    r_ref = op.residual(u).clone()
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    outs = []
    for i in range(12):
        with torch.cuda.stream(s1 if i % 2 == 0 else s2):
            o = torch.empty_like(u)
            op.jvp(u, v, out=o)
            rr = op.residual(u)
            outs.append((o, rr))
    torch.cuda.synchronize()
    for o, rr in outs:
        assert torch.equal(o, ref) and torch.equal(rr, r_ref)
