"""GPU parity: libfeod (CUDA, through the C-ABI) vs the CPU oracle.

Bar (BASELINE.json north_star): relative L2 error <= 1e-11 in fp64 on the same
seeded inputs, for r = F(u), J(u)v and the design gradient g.
Full vectors at reduced sizes spanning several bricks with ragged tails; the
full BASELINE sizes are covered by sampled rows in test_gpu_fullsize.py.
"""
import dataclasses

import numpy as np
import pytest

import oracle as O
import workloads as W
from gpu_util import rel_l2, problem, operator, cuda, host

pytestmark = pytest.mark.gpu
TOL = 1e-11

# (recipe, reduced n): n chosen so the mesh spans several bricks with a ragged last brick;
# the last four cases also span two brick slabs in z (BZ = 16, Q6: 8), so every fix-up set
# (x-, y- and z-faces, edges, corners) is exercised on full vectors
# Q6 on affine meshes with the kappa(u) models (9 stored values per point, rho for HEAT):
# the tensor-core path's general branches (C4 itself is the p-Laplacian)
Q6_NL = dataclasses.replace(W.C3, k=6, q=7, perturbed=False)
Q6_HEAT = dataclasses.replace(W.C5, k=6, q=7)
CASES = [(W.C1, 4), (W.C1, 7), (W.C2, 11), (W.C3, 6), (W.C3, 5), (W.C4, 3), (W.C5, 6), (W.C5, 9),
         (W.C3, 18), (W.C5, 17), (W.C2, 19), (W.C4, 9), (Q6_NL, 3), (Q6_HEAT, 2)]


def _case(w, n):
    ww = w.resized(n) if n != w.n else w
    return ww, W.draw(ww)


@pytest.mark.parametrize("w,n", CASES, ids=[f"{w.name}n{n}" for w, n in CASES])
def test_residual_parity(w, n):
    ww, d = _case(w, n)
    pr, op = problem(ww, d), operator(ww, d)
    r_ref = O.residual(pr, d["u"])
    r = host(op.residual(cuda(d["u"])))
    assert rel_l2(r, r_ref) <= TOL


@pytest.mark.parametrize("w,n", CASES, ids=[f"{w.name}n{n}" for w, n in CASES])
def test_jvp_parity(w, n):
    ww, d = _case(w, n)
    pr, op = problem(ww, d), operator(ww, d)
    Jv_ref = O.jvp(pr, d["u"], d["v"])
    Jv = host(op.jvp(cuda(d["u"]), cuda(d["v"])))
    assert rel_l2(Jv, Jv_ref) <= TOL
    r, Jv2 = op.jvp_res(cuda(d["u"]), cuda(d["v"]))
    assert rel_l2(host(Jv2), Jv_ref) <= TOL
    assert rel_l2(host(r), O.residual(pr, d["u"])) <= TOL


@pytest.mark.parametrize("n", [6, 9])
def test_design_grad_parity(n):
    ww, d = _case(W.C5, n)
    pr, op = problem(ww, d), operator(ww, d)
    g_ref = O.design_grad(pr, d["u"], d["lam"])
    g = host(op.design_grad(cuda(d["u"]), cuda(d["lam"])))
    assert rel_l2(g, g_ref) <= TOL


RG_CASES = [(W.C5, 6), (W.C5, 9), (W.C5, 17), (dataclasses.replace(W.C5, k=1, q=2, perturbed=True), 11),
            (dataclasses.replace(W.C5, k=3, q=4), 5)]


@pytest.mark.parametrize("w,n", RG_CASES, ids=[f"Q{w.k}n{n}" for w, n in RG_CASES])
def test_res_design_grad_parity(w, n):
    """feod_res_design_grad (SURVEY §8(b) fused r + g; one dual pass on Q1/Q2, the two
    calls on Q3+) against the oracle's Eq. 1 residual and design gradient."""
    ww, d = _case(w, n)
    pr, op = problem(ww, d), operator(ww, d)
    r, g = op.res_design_grad(cuda(d["u"]), cuda(d["lam"]))
    assert rel_l2(host(r), O.residual(pr, d["u"])) <= TOL
    assert rel_l2(host(g), O.design_grad(pr, d["u"], d["lam"])) <= TOL


@pytest.mark.parametrize("w,n", CASES, ids=[f"{w.name}n{n}" for w, n in CASES])
def test_vjp_parity(w, n):
    """J(u)^T w (NEXT-1) against the oracle's transposed Eq. 2; w = the recipe's v draw."""
    ww, d = _case(w, n)
    pr, op = problem(ww, d), operator(ww, d)
    ref = O.vjp(pr, d["u"], d["v"])
    got = host(op.vjp(cuda(d["u"]), cuda(d["v"])))
    assert rel_l2(got, ref) <= TOL


@pytest.mark.parametrize("w,n", CASES, ids=[f"{w.name}n{n}" for w, n in CASES])
def test_linearize_and_jvp_lin_parity(w, n):
    """NEXT-2: feod_linearize returns F(u) and stores D's linearisation; feod_jvp_lin
    applies J(u) from it alone. Both against the oracle's Eq. 1 / Eq. 2."""
    ww, d = _case(w, n)
    pr, op = problem(ww, d), operator(ww, d)
    r = host(op.linearize(cuda(d["u"])))
    assert rel_l2(r, O.residual(pr, d["u"])) <= TOL
    Jv = host(op.jvp_lin(cuda(d["v"])))
    assert rel_l2(Jv, O.jvp(pr, d["u"], d["v"])) <= TOL


# Q4 (thread-per-plane path, odd point count) and Q5 (the colour sweep), perturbed
Q4_NL = dataclasses.replace(W.C3, k=4, q=5)
Q5_PL = dataclasses.replace(W.C2, k=5, q=6)
DIAG_CASES = [(W.C1, 4), (W.C2, 11), (W.C3, 5), (W.C4, 3), (W.C5, 6), (W.C5, 9), (Q6_NL, 3), (Q6_HEAT, 2),
              (Q4_NL, 3), (Q5_PL, 2)]


@pytest.mark.parametrize("w,n", DIAG_CASES, ids=[f"{w.name}n{n}" for w, n in DIAG_CASES])
def test_jacobi_diag_parity(w, n):
    """NEXT-3: feod_jacobi_diag (sum-factorised, colour-assembled diagonal of the stored
    linearisation) against the oracle's scattered Eq. 3 element-tangent diagonal."""
    ww, d = _case(w, n)
    pr, op = problem(ww, d), operator(ww, d)
    op.linearize(cuda(d["u"]))
    got = host(op.jacobi_diag())
    assert rel_l2(got, O.jacobi_diag(pr, d["u"])) <= TOL


# Q4..Q6 (elemat_hi.cu tiled RES, elm.cu with global tangent scratch): perturbed Q4 with
# kappa(u), Q5 p-Laplacian, Q6 affine p-Laplacian (C4) and HEAT (rho, b = dFh/du)
Q4_PL_PERT = dataclasses.replace(W.C2, k=4, q=5)
EM_CASES = [(W.C1, 3), (W.C2, 5), (W.C3, 3), (W.C5, 3), (Q4_NL, 2), (Q4_PL_PERT, 2), (Q5_PL, 2), (W.C4, 2),
            (Q6_HEAT, 2)]


@pytest.mark.parametrize("elm", [False, True], ids=["RES", "ELM"])
@pytest.mark.parametrize("w,n", EM_CASES, ids=[f"{w.name}n{n}" for w, n in EM_CASES])
def test_element_matrices_parity(w, n, elm):
    """NEXT-4 (Table-1 analogue): element tangents K_e = B^T J_D B on the FP64 tensor
    cores, RES and ELM, against the oracle's Eq. 3 element tangents."""
    ww, d = _case(w, n)
    pr, op = problem(ww, d), operator(ww, d)
    E = ww.n_elems
    e0, ne = (1, E - 2) if E > 4 else (0, E)
    if ww.k >= 4:   # K_e is up to 941 KB per element: a ragged range of a few elements
        e0, ne = 1, min(E - 1, 5)
    got = host(op.element_matrices(cuda(d["u"]), e0, ne, elm=elm))
    ref = O.element_tangent(pr, d["u"], np.arange(e0, e0 + ne))
    assert rel_l2(got.ravel(), ref.ravel()) <= TOL
