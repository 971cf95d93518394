"""Pins T4-T14 and the Newton-CG driver for the CPU oracle.

Every expected value here comes from somewhere other than the oracle's own
formulas: closed forms (tests/golden/load_sums.json), Kronecker products of
exact 1D matrices built with numpy.polynomial, central finite differences,
the patch test, the Euler identity of the rho^3-homogeneous flux, brute-force
dense Jacobians, and a dense linear solve.
"""
import json
import os

import numpy as np
import pytest
from numpy.polynomial import polynomial as Pl

import oracle as O
from oracle import fem as F
import workloads as W

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "load_sums.json")))
PL, NL, HT = 0, 1, 2


def prob(n, k, model=PL, perturbed=False, faces=63, f=1.0, p=2.0, eps=0.0, rho=None, q=None):
    nx, ny, nz = (n, n, n) if np.isscalar(n) else n
    verts = None
    if perturbed:
        assert nx == ny == nz
        verts = W.vertices(nx, True)
    return O.Problem(nx, ny, nz, k, q or k + 1, model, p, eps, f, faces, verts, rho)


def rand_free(pr, seed, scale=1.0):
    x = scale * np.random.default_rng(seed).uniform(-1, 1, pr.n_dofs)
    x[O.dirichlet_mask(pr)] = 0.0
    return x


# ------------------------------------------------------------------ exact 1D matrices (T7)
def mat1d(k):
    """Exact element mass/stiffness on [0,1] for GLL cardinal functions (numpy.polynomial)."""
    if k == 1:
        return np.array([[1 / 3, 1 / 6], [1 / 6, 1 / 3]]), np.array([[1.0, -1.0], [-1.0, 1.0]])
    if k == 2:   # nodes 0, 1/2, 1
        M = np.array([[4, 2, -1], [2, 16, 2], [-1, 2, 4]]) / 30.0
        K = np.array([[7, -8, 1], [-8, 16, -8], [1, -8, 7]]) / 3.0
        return M, K
    nodes, _ = O.gll_nodes01(k)   # pinned by T2
    # exact for degree 2k: a (k+2)-point Gauss rule from numpy, cardinal functions in product form
    t, w = np.polynomial.legendre.leggauss(k + 2)
    x, w = (1 + t) / 2, w / 2
    V = np.ones((len(x), k + 1))
    Dv = np.zeros((len(x), k + 1))
    for a in range(k + 1):
        others = np.delete(nodes, a)
        den = np.prod(nodes[a] - others)
        V[:, a] = np.prod(x[:, None] - others[None, :], axis=1) / den
        for m in range(k):
            Dv[:, a] += np.prod(np.delete(x[:, None] - others[None, :], m, axis=1), axis=1) / den
    M = V.T @ (w[:, None] * V)
    K = Dv.T @ (w[:, None] * Dv)
    return M, K


def global1d(n, k):
    Me, Ke = mat1d(k)
    h = 1.0 / n
    m = k * n + 1
    M = np.zeros((m, m))
    K = np.zeros((m, m))
    for e in range(n):
        s = slice(k * e, k * e + k + 1)
        M[s, s] += h * Me
        K[s, s] += Ke / h
    return M, K


def kron_stiffness(nx, ny, nz, k):
    Mx, Kx = global1d(nx, k)
    My, Ky = global1d(ny, k)
    Mz, Kz = global1d(nz, k)
    K = np.kron(Mz, np.kron(My, Kx)) + np.kron(Mz, np.kron(Ky, Mx)) + np.kron(Kz, np.kron(My, Mx))
    b = np.kron(Mz.sum(1), np.kron(My.sum(1), Mx.sum(1)))
    return K, b


def test_mat1d_self_consistency():
    for k in (1, 2, 3, 4, 6):
        M, K = mat1d(k)
        assert abs(M.sum() - 1.0) < 1e-13
        np.testing.assert_allclose(K.sum(1), 0.0, atol=1e-10)
        np.testing.assert_allclose(M, M.T, atol=1e-14)
    # Q2 closed form vs the polynomial route
    nodes = np.array([0, 0.5, 1.0])
    cs = [Pl.polyfit(nodes, np.eye(3)[a], 2) for a in range(3)]
    m = Pl.polyint(Pl.polymul(cs[0], cs[1]))
    assert abs(Pl.polyval(1.0, m) - 2 / 30) < 1e-14


# ------------------------------------------------------------------ T4, T5
@pytest.mark.parametrize("k", [1, 2, 3])
def test_t4_volume_perturbed(k):
    pr = prob(4, k, perturbed=True)
    ch = F._Elements(pr, np.arange(pr.n_elems))
    assert abs(ch.W.sum() - 1.0) < 1e-13
    assert np.all(ch.detJ > 0)
    pa = prob(3, k)
    ch = F._Elements(pa, np.arange(pa.n_elems))
    np.testing.assert_allclose(ch.detJ, (1 / 3) ** 3, rtol=1e-13)


@pytest.mark.parametrize("k", [1, 2, 3])
def test_t5_gather_scatter_adjoint_and_map(k):
    pr = prob(3, k, perturbed=True)
    rng = np.random.default_rng(0)
    x = rng.standard_normal(pr.n_dofs)
    dofs = O.dof_map(pr)
    y = rng.standard_normal(dofs.shape)
    lhs = np.sum(x[dofs] * y)
    rhs = x @ np.bincount(dofs.ravel(), y.ravel(), minlength=pr.n_dofs)
    assert abs(lhs - rhs) < 1e-12 * abs(lhs)
    # every global DOF is reached; the map agrees with the node coordinates built
    # independently in workloads.node_coords (trilinear images of GLL nodes)
    assert len(np.unique(dofs)) == pr.n_dofs
    nodes, _ = O.gll_nodes01(k)
    X = W.node_coords(3, k, True, nodes)
    Phi, _, _, _ = F.tables(k, k + 1)
    # element (0,0,0) local node (a,b,c) must sit at the trilinear image of (xi_a, xi_b, xi_c)
    Xg = pr.vertex_grid()
    for c in range(k + 1):
        for b in range(k + 1):
            for a in range(k + 1):
                xi = np.array([nodes[a], nodes[b], nodes[c]])
                acc = sum(((xi[0] if dx else 1 - xi[0]) * (xi[1] if dy else 1 - xi[1]) *
                           (xi[2] if dz else 1 - xi[2])) * Xg[dz, dy, dx]
                          for dz in (0, 1) for dy in (0, 1) for dx in (0, 1))
                np.testing.assert_allclose(X[dofs[0, a + (k + 1) * (b + (k + 1) * c)]], acc, atol=1e-15)


# ------------------------------------------------------------------ T6 load
@pytest.mark.parametrize("case", [c for c in GOLD["cases"] if c["n"] <= 4])
def test_t6_load_sum_golden(case):
    pr = prob(case["n"], case["k"], faces=case["faces"], f=1.0, p=3.0, eps=1e-2)
    b = -O.residual(pr, np.zeros(pr.n_dofs))
    assert abs(b.sum() - case["value"]) < 1e-13
    assert abs(eval(case["expr"]) - case["value"]) < 1e-15


@pytest.mark.parametrize("model", [PL, NL, HT])
def test_t6_load_total_and_models(model):
    n, k = 3, 2
    rho = np.random.default_rng(1).uniform(0.1, 1, n ** 3)
    for faces, expect in ((0, 1.0), (1, 1 - (1 / 3) / 6)):
        pr = prob(n, k, model=model, perturbed=True, faces=faces, f=1.0, p=3.0, eps=1e-2, rho=rho)
        b = -O.residual(pr, np.zeros(pr.n_dofs))
        # the perturbation vanishes on the boundary, so the x=0 face load is unchanged
        assert abs(b.sum() - expect) < 1e-13


# ------------------------------------------------------------------ T7 p = 2 Kronecker
@pytest.mark.parametrize("dims,k", [((3, 3, 3), 1), ((2, 2, 2), 2), ((2, 3, 1), 2), ((2, 2, 2), 3),
                                    ((1, 1, 1), 6), ((2, 1, 2), 4)])
def test_t7_p2_kronecker(dims, k):
    pr = O.Problem(*dims, k, k + 1, PL, 2.0, 0.0, 1.0, 63)
    K, b = kron_stiffness(*dims, k)
    u = rand_free(pr, 7)
    u[O.dirichlet_mask(pr)] = np.random.default_rng(8).uniform(-1, 1, O.dirichlet_mask(pr).sum())
    r = O.residual(pr, u)
    expect = K @ u - b
    expect[O.dirichlet_mask(pr)] = 0.0
    assert np.linalg.norm(r - expect) <= 1e-12 * np.linalg.norm(expect)


# ------------------------------------------------------------------ T8 J(0)
@pytest.mark.parametrize("model,scale", [(PL, 1e-2), (NL, 1.0), (HT, 0.4 ** 3)])
def test_t8_jacobian_at_zero(model, scale):
    dims, k = (2, 2, 2), 2
    pr = O.Problem(*dims, k, k + 1, model, 3.0, 1e-2, 1.0, 63, None, np.full(8, 0.4))
    K, _ = kron_stiffness(*dims, k)
    v = np.random.default_rng(3).uniform(-1, 1, pr.n_dofs)
    Jv = O.jvp(pr, np.zeros(pr.n_dofs), v)
    expect = scale * (K @ v)
    expect[O.dirichlet_mask(pr)] = 0.0
    assert np.linalg.norm(Jv - expect) <= 1e-12 * np.linalg.norm(expect)


# ------------------------------------------------------------------ T9 patch test
@pytest.mark.parametrize("k", [1, 2, 3])
@pytest.mark.parametrize("perturbed", [False, True])
def test_t9_patch(k, perturbed):
    n = 3
    pr = prob(n, k, perturbed=perturbed, f=0.0, p=3.0, eps=1e-2)
    nodes, _ = O.gll_nodes01(k)
    X = W.node_coords(n, k, perturbed, nodes)
    u = X @ np.array([0.3, -0.7, 0.45]) + 0.2
    r = O.residual(pr, u)
    free = ~O.dirichlet_mask(pr)
    # scale: the un-cancelled element contributions
    parts = F._residual_elems(pr, u)
    scale = np.linalg.norm(np.bincount(parts[0][0].ravel(), np.abs(parts[0][1]).ravel(), pr.n_dofs))
    assert scale > 1e-3
    assert np.linalg.norm(r[free]) <= 1e-12 * scale
    # u = const gives r = 0 for every model with f = 0
    rho = np.full(pr.n_elems, 0.7)
    for model in (PL, NL, HT):
        prm = prob(n, k, model=model, perturbed=perturbed, f=0.0, p=3.0, eps=1e-2, rho=rho)
        assert np.max(np.abs(O.residual(prm, np.full(pr.n_dofs, 0.37)))) < 1e-14


# ------------------------------------------------------------------ T10 symmetry
@pytest.mark.parametrize("k,perturbed,p", [(1, True, 4.0), (2, True, 3.0), (3, False, 3.0)])
def test_t10_symmetry_plaplace(k, perturbed, p):
    pr = prob(3, k, perturbed=perturbed, p=p, eps=1e-2)
    u = rand_free(pr, 1)
    x, y = rand_free(pr, 2), rand_free(pr, 3)
    a, b = x @ O.jvp(pr, u, y), y @ O.jvp(pr, u, x)
    assert abs(a - b) <= 1e-12 * abs(a)


def test_t10_nonsymmetric_nldiff_and_const():
    pr = prob(3, 2, model=NL, perturbed=True)
    x, y = rand_free(pr, 2), rand_free(pr, 3)
    u = rand_free(pr, 1)
    a, b = x @ O.jvp(pr, u, y), y @ O.jvp(pr, u, x)
    assert abs(a - b) > 1e-6 * abs(a)          # reading A10: not symmetric in general
    c = np.full(pr.n_dofs, 0.6)
    a, b = x @ O.jvp(pr, c, y), y @ O.jvp(pr, c, x)
    assert abs(a - b) <= 1e-12 * abs(a)        # symmetric where grad u = 0


# ------------------------------------------------------------------ T11 pointwise J_D
def test_t11_pointwise():
    g = np.array([[1.0, 0.0, 0.0]])
    U = np.zeros(1)
    np.testing.assert_allclose(O.flux_dg(PL, U, g, p=3.0, eps=0.0)[0], np.diag([2.0, 1.0, 1.0]), atol=1e-15)
    np.testing.assert_allclose(O.flux_dg(PL, U, 0 * g, p=3.0, eps=1e-2)[0], 1e-2 * np.eye(3), atol=1e-15)
    np.testing.assert_allclose(O.flux_dg(PL, U, 0 * g, p=4.0, eps=1e-3)[0], 1e-6 * np.eye(3), atol=1e-18)
    np.testing.assert_allclose(O.flux_dg(PL, U, g, p=2.0)[0], np.eye(3), atol=0)
    rng = np.random.default_rng(5)
    for model in (PL, NL, HT):
        for _ in range(5):
            g = rng.standard_normal((1, 3))
            U = rng.standard_normal(1)
            kw = dict(p=rng.choice([2.0, 3.0, 4.0, 3.5]), eps=1e-2, rho=np.array([0.6]))
            Jg = O.flux_dg(model, U, g, **kw)[0]
            h = 1e-6
            fd = np.stack([(O.flux(model, U, g + h * e, **kw) - O.flux(model, U, g - h * e, **kw))[0] / (2 * h)
                           for e in np.eye(3)], axis=1)
            np.testing.assert_allclose(Jg, fd, rtol=1e-6, atol=1e-8)
            fdu = (O.flux(model, U + h, g, **kw) - O.flux(model, U - h, g, **kw))[0] / (2 * h)
            np.testing.assert_allclose(O.flux_du(model, U, g, **kw)[0], fdu, rtol=1e-6, atol=1e-8)
            kr = dict(kw)
            fr = []
            for s in (1, -1):
                kr["rho"] = kw["rho"] + s * h
                fr.append(O.flux(model, U, g, **kr)[0])
            np.testing.assert_allclose(O.flux_drho(model, U, g, **kw)[0], (fr[0] - fr[1]) / (2 * h),
                                       rtol=1e-6, atol=1e-8)
            assert np.min(np.linalg.eigvalsh((Jg + Jg.T) / 2)) > 0    # PSD (and monotone)
            np.testing.assert_allclose(Jg, Jg.T, atol=1e-14)
            # rotation equivariance: D(R g) = R D(g)
            Rq, _ = np.linalg.qr(rng.standard_normal((3, 3)))
            np.testing.assert_allclose(O.flux(model, U, g @ Rq.T, **kw), O.flux(model, U, g, **kw) @ Rq.T,
                                       rtol=1e-13, atol=1e-14)


# ------------------------------------------------------------------ T12 Taylor
@pytest.mark.parametrize("model,k,perturbed", [(PL, 2, True), (NL, 3, True), (HT, 2, False)])
def test_t12_taylor(model, k, perturbed):
    rho = np.random.default_rng(9).uniform(0.1, 1, 27)
    pr = prob(3, k, model=model, perturbed=perturbed, faces=63 if model != HT else 1,
              p=3.0, eps=1e-2, rho=rho)
    u, v = rand_free(pr, 1), np.random.default_rng(2).uniform(-1, 1, pr.n_dofs)
    F0, Jv = O.residual(pr, u), O.jvp(pr, u, v)
    errs = [np.linalg.norm(O.residual(pr, u + h * v) - F0 - h * Jv) for h in (1e-1, 5e-2, 2.5e-2, 1.25e-2)]
    rates = [np.log2(errs[i] / errs[i + 1]) for i in range(3)]
    assert all(abs(r - 2) < 0.1 for r in rates), rates
    h = 1e-5
    cd = (O.residual(pr, u + h * v) - O.residual(pr, u - h * v)) / (2 * h)
    assert np.linalg.norm(cd - Jv) <= 1e-7 * np.linalg.norm(Jv)


# ------------------------------------------------------------------ T13 dense brute force
CASES13 = [
    dict(n=2, k=2, model=PL, perturbed=False, faces=63, p=3.0, eps=1e-2),
    dict(n=1, k=6, model=PL, perturbed=False, faces=63, p=3.0, eps=1e-2),
    dict(n=3, k=1, model=PL, perturbed=True, faces=63, p=4.0, eps=1e-3),
    dict(n=2, k=2, model=HT, perturbed=False, faces=1, p=2.0, eps=0.0),
    dict(n=2, k=3, model=NL, perturbed=True, faces=63, p=2.0, eps=0.0),
    # Q4 / Q5 element tangents (the K9b / ELM orders) pinned the same way
    dict(n=1, k=4, model=NL, perturbed=True, faces=1, p=2.0, eps=0.0),
    dict(n=1, k=5, model=PL, perturbed=True, faces=2, p=3.0, eps=1e-2),
]


@pytest.mark.parametrize("c", CASES13, ids=lambda c: f"n{c['n']}k{c['k']}m{c['model']}")
def test_t13_dense_jacobian(c):
    n = c["n"]
    rho = np.random.default_rng(4).uniform(0.1, 1, n ** 3)
    pr = prob(n, c["k"], model=c["model"], perturbed=c["perturbed"], faces=c["faces"],
              p=c["p"], eps=c["eps"], rho=rho)
    u = rand_free(pr, 11)
    A = O.dense_jacobian(pr, u)
    N = pr.n_dofs
    cols = np.stack([O.jvp(pr, u, e) for e in np.eye(N)], axis=1)
    assert np.max(np.abs(A - cols)) <= 1e-12 * np.max(np.abs(A))
    free = np.flatnonzero(~O.dirichlet_mask(pr))
    pick = free if len(free) <= 40 else free[:: max(1, len(free) // 40)]
    h = 1e-6
    for j in pick:
        e = np.zeros(N)
        e[j] = 1.0
        fd = (O.residual(pr, u + h * e) - O.residual(pr, u - h * e)) / (2 * h)
        assert np.max(np.abs(fd - A[:, j])) <= 1e-7 * max(1.0, np.max(np.abs(A)))
    # a Dirichlet column enters the free rows (reading A2)
    d = np.flatnonzero(O.dirichlet_mask(pr))[len(free) % 7]
    e = np.zeros(N)
    e[d] = 1.0
    fd = (O.residual(pr, u + h * e) - O.residual(pr, u - h * e)) / (2 * h)
    assert np.max(np.abs(fd - A[:, d])) <= 1e-7 * max(1.0, np.max(np.abs(A)))


# ------------------------------------------------------------------ T14 design gradient
def test_t14_design_gradient():
    n, k = 3, 2
    rng = np.random.default_rng(21)
    rho = rng.uniform(0.1, 1, n ** 3)
    pr = prob(n, k, model=HT, perturbed=True, faces=1, f=1.0, rho=rho)
    u, lam = rng.uniform(-1, 1, pr.n_dofs), rng.uniform(-1, 1, pr.n_dofs)
    mask = O.dirichlet_mask(pr)
    u[mask] = 0.0
    g = O.design_grad(pr, u, lam)
    lm = lam.copy()
    lm[mask] = 0.0
    # (i) central FD in rho_e of -lambda^T F (free rows)
    h = 1e-6
    for e in (0, 5, 13, 26):
        rp, rm = rho.copy(), rho.copy()
        rp[e] += h
        rm[e] -= h
        fp = O.residual(O.Problem(**{**pr.__dict__, "rho": rp}), u)
        fm = O.residual(O.Problem(**{**pr.__dict__, "rho": rm}), u)
        assert abs(-(lm @ (fp - fm)) / (2 * h) - g[e]) <= 1e-7 * np.max(np.abs(g))
    # (ii) Euler identity: sum rho_e g_e = -3 lambda^T (F(u) + b), b = -F(0)
    Fu, F0 = O.residual(pr, u), O.residual(pr, np.zeros_like(u))
    lhs, rhs = rho @ g, -3.0 * (lm @ (Fu - F0))
    assert abs(lhs - rhs) <= 1e-12 * np.sum(np.abs(rho * g))
    # (iii) degree-2 homogeneity of g in rho
    g2 = O.design_grad(O.Problem(**{**pr.__dict__, "rho": 1.7 * rho}), u, lam)
    np.testing.assert_allclose(g2, 1.7 ** 2 * g, rtol=1e-12, atol=1e-15)
    # (iv) independent of f;  (v) u = const gives g = 0
    g3 = O.design_grad(O.Problem(**{**pr.__dict__, "f": 5.0}), u, lam)
    np.testing.assert_array_equal(g3, g)
    assert np.max(np.abs(O.design_grad(pr, np.full_like(u, 0.3), lam))) < 1e-15
    # only free rows of lambda count
    lam2 = lam.copy()
    lam2[mask] = 123.0
    np.testing.assert_array_equal(O.design_grad(pr, u, lam2), g)


# ------------------------------------------------------------------ sampled rows
def test_sampled_rows_match_full():
    pr = prob(4, 2, model=NL, perturbed=True)
    u, v = rand_free(pr, 1), rand_free(pr, 2)
    rows = np.random.default_rng(3).choice(pr.n_dofs, 50, replace=False)
    np.testing.assert_allclose(O.residual_rows(pr, u, rows), O.residual(pr, u)[rows], rtol=1e-14, atol=1e-16)
    np.testing.assert_allclose(O.jvp_rows(pr, u, v, rows), O.jvp(pr, u, v)[rows], rtol=1e-14, atol=1e-16)


# ------------------------------------------------------------------ Newton-CG driver
def test_cg_fixed_dense():
    from oracle.newton import cg_fixed
    rng = np.random.default_rng(0)
    A = rng.standard_normal((12, 12))
    A = A @ A.T + 12 * np.eye(12)
    b = rng.standard_normal(12)
    x, _ = cg_fixed(lambda y: A @ y, b, 12)
    np.testing.assert_allclose(x, np.linalg.solve(A, b), rtol=1e-10)
    x1, _ = cg_fixed(lambda y: 2.0 * y, b, 1)       # A = 2I converges in one iteration
    np.testing.assert_allclose(x1, b / 2, rtol=1e-15)


def test_newton_cg_linear_case():
    # p = 2: one Newton step with enough CG iterations solves K u = b exactly
    pr = O.Problem(2, 2, 2, 2, 3, PL, 2.0, 0.0, 1.0, 63)
    K, b = kron_stiffness(2, 2, 2, 2)
    free = ~O.dirichlet_mask(pr)
    u, norms = O.newton_cg(pr, np.zeros(pr.n_dofs), newton_steps=1, cg_iters=int(free.sum()))
    exact = np.zeros(pr.n_dofs)
    exact[free] = np.linalg.solve(K[np.ix_(free, free)], b[free])
    np.testing.assert_allclose(u, exact, rtol=1e-10, atol=1e-14)
    assert norms[-1] < 1e-12 * norms[0]


# ------------------------------------------------------------------ T15 transposed Jacobian (NEXT-1)
@pytest.mark.parametrize("c", CASES13, ids=lambda c: f"n{c['n']}k{c['k']}m{c['model']}")
def test_t15_vjp_is_transposed_dense_jacobian(c):
    """J^T w against the transpose of the dense Jacobian that T13 pins to central
    finite differences of the residual, and the adjoint identity <w, J v> = <J^T w, v>
    against the (separately pinned) JVP."""
    n = c["n"]
    rho = np.random.default_rng(4).uniform(0.1, 1, n ** 3)
    pr = prob(n, c["k"], model=c["model"], perturbed=c["perturbed"], faces=c["faces"],
              p=c["p"], eps=c["eps"], rho=rho)
    u = rand_free(pr, 11)
    rng = np.random.default_rng(12)
    w, v = rng.uniform(-1, 1, pr.n_dofs), rng.uniform(-1, 1, pr.n_dofs)
    A = O.dense_jacobian(pr, u)
    JTw = O.vjp(pr, u, w)
    np.testing.assert_allclose(JTw, A.T @ w, rtol=0, atol=1e-12 * np.max(np.abs(A)) * np.abs(w).sum())
    lhs, rhs = w @ O.jvp(pr, u, v), JTw @ v
    assert abs(lhs - rhs) <= 1e-12 * (np.abs(w) @ np.abs(A) @ np.abs(v))
    # w's Dirichlet entries do not matter
    w2 = w.copy()
    w2[O.dirichlet_mask(pr)] = 7.0
    np.testing.assert_array_equal(O.vjp(pr, u, w2), JTw)


def test_t16_adjoint_solve_dense():
    """The dense adjoint solution satisfies (J^T lambda)_free = rhs_free through the
    separately pinned J^T w (T15), with lambda_Dir = 0 (heat model: nonsymmetric J)."""
    n, k = 3, 2
    rng = np.random.default_rng(31)
    rho = rng.uniform(0.1, 1, n ** 3)
    pr = prob(n, k, model=HT, perturbed=True, faces=1, f=1.0, rho=rho)
    u = rand_free(pr, 32)
    rhs = rng.uniform(-1, 1, pr.n_dofs)
    lam = O.adjoint_solve(pr, u, rhs)
    mask = O.dirichlet_mask(pr)
    assert np.all(lam[mask] == 0.0)
    res = O.vjp(pr, u, lam) - rhs
    assert np.linalg.norm(res[~mask]) <= 1e-10 * np.linalg.norm(rhs)
    A = O.dense_jacobian(pr, u)[np.ix_(~mask, ~mask)]
    assert np.max(np.abs(A - A.T)) > 1e-3 * np.max(np.abs(A))   # the free block is genuinely nonsymmetric


def test_bicgstab_fixed_solves_nonsymmetric():
    """Pin for the reference BiCGStab: on a nonsymmetric, diagonally dominant matrix
    it reaches numpy.linalg.solve's answer, and its recursive residual matches the
    true residual."""
    rng = np.random.default_rng(3)
    n = 60
    A = rng.uniform(-1, 1, (n, n)) + n * np.eye(n)
    b = rng.uniform(-1, 1, n)
    x, hist = O.bicgstab_fixed(lambda y: A @ y, b, 40)
    np.testing.assert_allclose(x, np.linalg.solve(A, b), rtol=0, atol=1e-12)
    assert hist[-1] <= 1e-12 * hist[0]
    x5, h5 = O.bicgstab_fixed(lambda y: A @ y, b, 5)
    assert abs(np.linalg.norm(b - A @ x5) - h5[-1]) <= 1e-10 * h5[0]


@pytest.mark.parametrize("c", CASES13, ids=lambda c: f"n{c['n']}k{c['k']}m{c['model']}")
def test_jacobi_diag_is_dense_diagonal(c):
    """NEXT-3: the scattered element-tangent diagonal equals the diagonal of the
    FD-pinned dense Jacobian (T13) on free rows, 1 on Dirichlet rows."""
    n = c["n"]
    rho = np.random.default_rng(4).uniform(0.1, 1, n ** 3)
    pr = prob(n, c["k"], model=c["model"], perturbed=c["perturbed"], faces=c["faces"],
              p=c["p"], eps=c["eps"], rho=rho)
    u = rand_free(pr, 11)
    d = O.jacobi_diag(pr, u)
    mask = O.dirichlet_mask(pr)
    A = O.dense_jacobian(pr, u)
    np.testing.assert_allclose(d[~mask], np.diag(A)[~mask], rtol=1e-13, atol=0)
    assert np.all(d[mask] == 1.0)


def test_pcg_fixed_reaches_solve():
    """Pin for the Jacobi-preconditioned CG: on a badly scaled SPD matrix it reaches
    numpy.linalg.solve's answer (and faster than plain CG)."""
    rng = np.random.default_rng(6)
    n = 50
    Q = rng.uniform(-1, 1, (n, n))
    S = np.diag(10.0 ** rng.uniform(-3, 3, n))
    A = S @ (Q @ Q.T + n * np.eye(n)) @ S
    b = rng.uniform(-1, 1, n)
    x, _ = O.cg_fixed(lambda y: A @ y, b, 60, np.diag(A).copy())
    np.testing.assert_allclose(x, np.linalg.solve(A, b), rtol=1e-9)
    x0, _ = O.cg_fixed(lambda y: A @ y, b, 60)
    assert np.linalg.norm(A @ x - b) < 1e-3 * np.linalg.norm(A @ x0 - b)


def test_vjp_rows_match_full():
    pr = prob(4, 2, model=HT, perturbed=True, faces=1, rho=np.random.default_rng(2).uniform(0.1, 1, 64))
    u, w = rand_free(pr, 1), np.random.default_rng(3).uniform(-1, 1, pr.n_dofs)
    rows = np.array([0, 5, 40, 100, pr.n_dofs - 1])
    np.testing.assert_array_equal(O.vjp_rows(pr, u, w, rows), O.vjp(pr, u, w)[rows])


# ------------------------------------------------------------------ reading A20 (eps = 0, grad u = 0)
@pytest.mark.parametrize("p", [2.5, 3.0, 3.5, 4.0])
def test_a20_eps0_zero_gradient_limit(p):
    """p-Laplacian with eps = 0 where grad u vanishes identically (u = 0 away from one
    node): the JVP is finite, exactly 0 on rows whose elements all have grad u = 0 (the
    limit of dD/dg ~ |g|^(p-2) -> 0), and central FD of the residual tends to it at the
    rate h^(p-2) (a wrong limit -- NaN, or k I with k != 0 -- fails)."""
    pr = prob(3, 2, PL, perturbed=False, p=p, eps=0.0)
    u = np.zeros(pr.n_dofs)
    m = 2 * 3 + 1
    c = 2 + m * (2 + m * 2)                 # an interior node: (2, 2, 2)
    u[c] = 1.0
    v = rand_free(pr, 5)
    Jv = O.jvp(pr, u, v)
    assert np.all(np.isfinite(Jv))
    # rows coupled to node c only through elements with grad u != 0
    hot = O.jvp(pr, u, np.where(np.arange(pr.n_dofs) == c, 1.0, 0.0)) != 0.0
    X = np.arange(pr.n_dofs) % m
    Y = (np.arange(pr.n_dofs) // m) % m
    Z = np.arange(pr.n_dofs) // (m * m)
    touched = (np.abs(X - 2) <= 2) & (np.abs(Y - 2) <= 2) & (np.abs(Z - 2) <= 2)   # rows of the elements at c
    cold = ~touched & ~O.dirichlet_mask(pr)
    assert cold.any() and hot.any()
    assert np.all(Jv[cold] == 0.0)
    F = lambda x: O.residual(pr, x)
    errs, errs_all = [], []
    for h in (1e-2, 1e-4):
        fd = (F(u + h * v) - F(u - h * v)) / (2 * h)
        errs.append(np.max(np.abs(fd[cold])))
        errs_all.append(np.max(np.abs(fd - Jv)))
    # FD on the cold rows decays like h^(p-2) to the limit 0 (h ratio 100); on all rows
    # the FD error decays at least that fast (second order where the flux is smooth)
    rate = 100.0 ** (-min(p - 2.0, 2.0))
    assert errs[1] <= errs[0] * rate * 4.0 + 1e-13
    assert errs_all[1] <= errs_all[0] * rate * 4.0 + 1e-12
    assert np.isfinite(errs_all).all() and errs_all[1] < errs_all[0]
