"""Dense, non-sum-factorised FEOD operators (test infrastructure only).

PAPER.md §2 (lines 25, 148-162): A_p(u) = P^T G^T B^T D(B G P u) (Eq. 1) and
J_p(u) = P^T G^T B^T J_D(u_q) B G P (Eq. 2), on hexahedral Q_k elements of a
structured unit-cube mesh (BASELINE.json north_star / configs).

Each operator is written out in the paper's order:
  P   -> readings A2 (Dirichlet rows) — full-length vectors, F_i = 0 on Dirichlet rows
  G   -> ``dof_map``: u_e = u[dofs_e]                                   (line 112-113)
  B   -> dense tables Phi, dPhi_d (q^3 x (k+1)^3) and the trilinear geometry
         J_q = dx/dxi, inverted with numpy.linalg.inv                   (line 126-127)
  D   -> oracle/flux.py, evaluated at the physical gradient J^{-T} dPhi u_e
  B^T -> dPhi_d^T (W (J^{-1} D)_d) - Phi^T (W f)   (the -div convention, A1)
  G^T -> numpy.bincount over the DOF map (fixed sequential order)
  P^T -> zero the Dirichlet rows.

Element order is x-fastest lexicographic e = ex + nx (ey + ny ez); DOF order is
x-fastest lexicographic over the (k nx + 1) x (k ny + 1) x (k nz + 1) grid (A16).
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np

from .rules import gauss_legendre01, gll_nodes01, lagrange_eval
from . import flux as fx

FACE_X0, FACE_X1, FACE_Y0, FACE_Y1, FACE_Z0, FACE_Z1 = 1, 2, 4, 8, 16, 32


@dataclasses.dataclass
class Problem:
    nx: int
    ny: int
    nz: int
    k: int
    q: int
    model: int = fx.PLAPLACE
    p: float = 2.0
    eps: float = 0.0
    f: float = 0.0
    faces: int = 63
    verts: Optional[np.ndarray] = None   # (nx+1)(ny+1)(nz+1) x 3, x-fastest; None = uniform grid
    rho: Optional[np.ndarray] = None     # (E,) element densities (HEAT)

    @classmethod
    def from_workload(cls, w, verts=None, rho=None):
        return cls(w.n, w.n, w.n, w.k, w.q, w.model, w.p, w.eps, w.f, w.faces, verts, rho)

    @property
    def n_elems(self):
        return self.nx * self.ny * self.nz

    @property
    def dims(self):
        return (self.k * self.nx + 1, self.k * self.ny + 1, self.k * self.nz + 1)

    @property
    def n_dofs(self):
        a, b, c = self.dims
        return a * b * c

    def vertex_grid(self):
        if self.verts is not None:
            return np.asarray(self.verts, dtype=np.float64).reshape(self.nz + 1, self.ny + 1, self.nx + 1, 3)
        x = np.arange(self.nx + 1) / self.nx
        y = np.arange(self.ny + 1) / self.ny
        z = np.arange(self.nz + 1) / self.nz
        Z, Y, X = np.meshgrid(z, y, x, indexing="ij")
        return np.stack([X, Y, Z], axis=-1)


# ----------------------------------------------------------------------------- tables
def tables(k: int, q: int):
    """Dense 3D tables: Phi[qp, node], dPhi[d][qp, node], weights w[qp].

    qp = i + q (j + q l) (x fastest), node = a + (k+1)(b + (k+1) c).
    Phi = l_a(x_i) l_b(x_j) l_c(x_l); dPhi_1 = l_a' l_b l_c, etc.
    """
    nodes, _ = gll_nodes01(k)
    pts, wts = gauss_legendre01(q)
    V, D = lagrange_eval(nodes, pts)
    nd = k + 1

    def t3(A, B, C):
        return np.einsum("ia,jb,lc->ljicba", A, B, C).reshape(q ** 3, nd ** 3)

    Phi = t3(V, V, V)
    dPhi = [t3(D, V, V), t3(V, D, V), t3(V, V, D)]
    w = np.einsum("i,j,l->lji", wts, wts, wts).reshape(-1)
    return Phi, dPhi, w, pts


def dof_map(pr: Problem, elems=None):
    """G: (E, (k+1)^3) global DOF index of every local node (line 112-113)."""
    k, nd = pr.k, pr.k + 1
    Mx, My, _ = pr.dims
    if elems is None:
        elems = np.arange(pr.n_elems)
    elems = np.asarray(elems)
    ex = elems % pr.nx
    ey = (elems // pr.nx) % pr.ny
    ez = elems // (pr.nx * pr.ny)
    a = np.arange(nd)
    C, B, A = np.meshgrid(a, a, a, indexing="ij")
    A, B, C = A.reshape(-1), B.reshape(-1), C.reshape(-1)
    I = k * ex[:, None] + A[None, :]
    J = k * ey[:, None] + B[None, :]
    K = k * ez[:, None] + C[None, :]
    return I + Mx * (J + My * K)


def dirichlet_mask(pr: Problem):
    """Boolean mask of DOFs on the flagged faces (reading A2)."""
    Mx, My, Mz = pr.dims
    K, J, I = np.meshgrid(np.arange(Mz), np.arange(My), np.arange(Mx), indexing="ij")
    m = np.zeros((Mz, My, Mx), dtype=bool)
    if pr.faces & FACE_X0: m |= I == 0
    if pr.faces & FACE_X1: m |= I == Mx - 1
    if pr.faces & FACE_Y0: m |= J == 0
    if pr.faces & FACE_Y1: m |= J == My - 1
    if pr.faces & FACE_Z0: m |= K == 0
    if pr.faces & FACE_Z1: m |= K == Mz - 1
    return m.reshape(-1)


def geometry(pr: Problem, elems, pts):
    """Per-point trilinear Jacobian J[e, qp, c, d] = dx_c / dxi_d, (E, q^3, 3, 3)."""
    Xg = pr.vertex_grid()
    elems = np.asarray(elems)
    ex = elems % pr.nx
    ey = (elems // pr.nx) % pr.ny
    ez = elems // (pr.nx * pr.ny)
    Xv = np.empty((len(elems), 2, 2, 2, 3))
    for dz in (0, 1):
        for dy in (0, 1):
            for dx in (0, 1):
                Xv[:, dz, dy, dx, :] = Xg[ez + dz, ey + dy, ex + dx]
    N = np.stack([1.0 - pts, pts], axis=1)            # (q, 2) vertex shape functions
    dN = np.stack([-np.ones_like(pts), np.ones_like(pts)], axis=1)
    q = len(pts)
    cols = [np.einsum("ezyxc,ix,jy,lz->eljic", Xv, dN, N, N),
            np.einsum("ezyxc,ix,jy,lz->eljic", Xv, N, dN, N),
            np.einsum("ezyxc,ix,jy,lz->eljic", Xv, N, N, dN)]
    J = np.stack(cols, axis=-1).reshape(len(elems), q ** 3, 3, 3)
    return J


class _Elements:
    """Everything B needs for a chunk of elements."""

    def __init__(self, pr: Problem, elems):
        self.pr = pr
        self.elems = np.asarray(elems)
        self.Phi, self.dPhi, self.w, pts = tables(pr.k, pr.q)
        self.dofs = dof_map(pr, self.elems)
        J = geometry(pr, self.elems, pts)
        self.detJ = np.linalg.det(J)
        if np.any(self.detJ <= 0):
            raise ValueError("inverted element")
        self.Jinv = np.linalg.inv(J)
        self.W = self.w[None, :] * self.detJ
        self.rho = None
        if pr.rho is not None:
            self.rho = np.asarray(pr.rho)[self.elems][:, None]

    def interp(self, x):
        """B: values (E, q^3) and physical gradients (E, q^3, 3) of the field x."""
        xe = x[self.dofs]
        U = xe @ self.Phi.T
        Gref = np.stack([xe @ d.T for d in self.dPhi], axis=-1)
        # grad u = J^{-T} grad_ref u:  g_c = sum_d Jinv[d, c] Gref_d
        g = np.einsum("eqdc,eqd->eqc", self.Jinv, Gref)
        return U, g

    def test_grad(self, Dphys):
        """B^T for a flux: r_e[node] = sum_q W (J^{-1} D)_d dPhi_d[q, node]."""
        JD = np.einsum("eqdc,eqc->eqd", self.Jinv, Dphys) * self.W[..., None]
        return sum(JD[..., d] @ self.dPhi[d] for d in range(3))

    def test_val(self, S):
        """B^T for a value channel: r_e[node] = sum_q W S Phi[q, node]."""
        return (self.W * S) @ self.Phi


def _chunks(pr: Problem, elems=None):
    if elems is None:
        elems = np.arange(pr.n_elems)
    step = max(16, 6_000_000 // (pr.q ** 3 * (pr.k + 1) ** 3 + 64 * pr.q ** 3))
    for s in range(0, len(elems), step):
        yield _Elements(pr, elems[s:s + step])


def _params(pr, ch):
    return dict(p=pr.p, eps=pr.eps, rho=ch.rho)


def _assemble(pr, parts, n):
    idx = np.concatenate([d.ravel() for d, _ in parts]) if parts else np.zeros(0, int)
    val = np.concatenate([v.ravel() for _, v in parts]) if parts else np.zeros(0)
    r = np.bincount(idx, weights=val, minlength=n)
    r[dirichlet_mask(pr)] = 0.0
    return r


# ----------------------------------------------------------------------------- operators
def _residual_elems(pr, u, elems=None):
    parts = []
    for ch in _chunks(pr, elems):
        U, g = ch.interp(u)
        D = fx.flux(pr.model, U, g, **_params(pr, ch))
        re = ch.test_grad(D) - ch.test_val(np.full_like(U, pr.f))
        parts.append((ch.dofs, re))
    return parts


def _jvp_elems(pr, u, v, elems=None):
    parts = []
    for ch in _chunks(pr, elems):
        U, g = ch.interp(u)
        V, gv = ch.interp(v)
        kw = _params(pr, ch)
        Ddot = (np.einsum("eqcd,eqd->eqc", fx.flux_dg(pr.model, U, g, **kw), gv)
                + fx.flux_du(pr.model, U, g, **kw) * V[..., None])
        parts.append((ch.dofs, ch.test_grad(Ddot)))
    return parts


def residual(pr: Problem, u):
    """Eq. 1: r = P^T G^T B^T D(B G P u), r_i = 0 on Dirichlet rows."""
    return _assemble(pr, _residual_elems(pr, np.asarray(u, dtype=np.float64)), pr.n_dofs)


def jvp(pr: Problem, u, v):
    """Eq. 2: J(u) v = P^T G^T B^T J_D(u_q) B G P v, (Jv)_i = 0 on Dirichlet rows."""
    return _assemble(pr, _jvp_elems(pr, np.asarray(u, float), np.asarray(v, float)), pr.n_dofs)


def _vjp_elems(pr, u, w, elems=None):
    w = np.array(w, dtype=np.float64)
    w[dirichlet_mask(pr)] = 0.0           # J has zero Dirichlet rows, so J^T drops w there (A2)
    parts = []
    for ch in _chunks(pr, elems):
        U, g = ch.interp(u)
        _, gw = ch.interp(w)
        kw = _params(pr, ch)
        # column j of J (Eq. 2): sum_q W grad phi_i . (Dg grad phi_j + Du phi_j); transposed:
        #   (J^T w)_j = sum_q W [(Dg^T grad w) . grad phi_j + (Du . grad w) phi_j]
        Gbar = np.einsum("eqcd,eqc->eqd", fx.flux_dg(pr.model, U, g, **kw), gw)
        Sbar = np.einsum("eqc,eqc->eq", fx.flux_du(pr.model, U, g, **kw), gw)
        parts.append((ch.dofs, ch.test_grad(Gbar) + ch.test_val(Sbar)))
    return parts


def vjp(pr: Problem, u, w):
    """Transpose of Eq. 2 (the adjoint of line 199):
    J(u)^T w = P^T G^T B^T J_D(u_q)^T B G (Z w), Z zeroing w's Dirichlet entries
    (the rows J drops, reading A2); every output row is kept (no P^T row mask)."""
    idx_val = _vjp_elems(pr, np.asarray(u, float), w)
    idx = np.concatenate([d.ravel() for d, _ in idx_val]) if idx_val else np.zeros(0, int)
    val = np.concatenate([v.ravel() for _, v in idx_val]) if idx_val else np.zeros(0)
    return np.bincount(idx, weights=val, minlength=pr.n_dofs)


def adjoint_solve(pr: Problem, u, rhs):
    """Dense reference for feod_adjoint_solve: lambda with lambda_Dir = 0 and
    (J(u)^T lambda)_f = rhs_f on the free rows f, i.e. the transpose of the
    free-free block of the Eq. 3 Jacobian, solved by numpy.linalg.solve."""
    A = dense_jacobian(pr, u)
    f = np.flatnonzero(~dirichlet_mask(pr))
    lam = np.zeros(pr.n_dofs)
    lam[f] = np.linalg.solve(A[np.ix_(f, f)].T, np.asarray(rhs, float)[f])
    return lam


def _design_elems(pr, u, lam, elems=None):
    lam = np.array(lam, dtype=np.float64)
    lam[dirichlet_mask(pr)] = 0.0         # only free rows count (reading A14)
    out = []
    for ch in _chunks(pr, elems):
        U, g = ch.interp(u)
        _, gl = ch.interp(lam)
        dD = fx.flux_drho(pr.model, U, g, **_params(pr, ch))
        out.append(-np.sum(ch.W * np.einsum("eqc,eqc->eq", dD, gl), axis=1))
    return np.concatenate(out) if out else np.zeros(0)


def design_grad(pr: Problem, u, lam):
    """Line 199 / reading A14: g_e = -sum_{i free} lam_i dF_i/drho_e, lexicographic e."""
    return _design_elems(pr, np.asarray(u, float), lam)


# ----------------------------------------------------------------------------- sampled outputs
def _elems_touching(pr: Problem, rows):
    Mx, My, _ = pr.dims
    rows = np.asarray(rows)
    I, J, K = rows % Mx, (rows // Mx) % My, rows // (Mx * My)
    out = []
    for ox in (0, 1):
        for oy in (0, 1):
            for oz in (0, 1):
                ex = (I - ox) // pr.k
                ey = (J - oy) // pr.k
                ez = (K - oz) // pr.k
                # the element must contain the node: k ex <= I <= k (ex+1)
                ok = ((ex >= 0) & (ex < pr.nx) & (ey >= 0) & (ey < pr.ny) & (ez >= 0) & (ez < pr.nz)
                      & (I - pr.k * ex <= pr.k) & (J - pr.k * ey <= pr.k) & (K - pr.k * ez <= pr.k))
                out.append((ex + pr.nx * (ey + pr.ny * ez))[ok])
    return np.unique(np.concatenate(out))


def residual_rows(pr: Problem, u, rows):
    """r[rows], from only the elements that touch those rows."""
    el = _elems_touching(pr, rows)
    return _assemble(pr, _residual_elems(pr, np.asarray(u, float), el), pr.n_dofs)[rows]


def jvp_rows(pr: Problem, u, v, rows):
    el = _elems_touching(pr, rows)
    return _assemble(pr, _jvp_elems(pr, np.asarray(u, float), np.asarray(v, float), el), pr.n_dofs)[rows]


def vjp_rows(pr: Problem, u, w, rows):
    """(J^T w)[rows], from only the elements that touch those rows (no row mask, A17)."""
    el = _elems_touching(pr, rows)
    parts = _vjp_elems(pr, np.asarray(u, float), w, el)
    idx = np.concatenate([d.ravel() for d, _ in parts])
    val = np.concatenate([v.ravel() for _, v in parts])
    return np.bincount(idx, weights=val, minlength=pr.n_dofs)[rows]


def design_grad_elems(pr: Problem, u, lam, elems):
    return _design_elems(pr, np.asarray(u, float), lam, np.asarray(elems))


# ----------------------------------------------------------------------------- Eq. 3 / dense
def element_tangent(pr: Problem, u, elems):
    """Eq. 3: K_e = B^T J_D(u_q) B, (E, nd^3, nd^3), K_e[i, j] = d r_e,i / d u_e,j."""
    u = np.asarray(u, float)
    out = []
    for ch in _chunks(pr, np.asarray(elems)):
        U, g = ch.interp(u)
        kw = _params(pr, ch)
        Dg = fx.flux_dg(pr.model, U, g, **kw)        # (E, Q, 3, 3)
        Du = fx.flux_du(pr.model, U, g, **kw)        # (E, Q, 3)
        gref = np.stack(ch.dPhi, axis=-1)             # (Q, nodes, 3)
        gphys = np.einsum("eqdc,qnd->eqnc", ch.Jinv, gref)   # physical grads of every phi
        # column j: Ddot = Dg grad phi_j + Du phi_j ; row i: sum_q W Ddot . grad phi_i
        Ddot = np.einsum("eqcd,eqjd->eqjc", Dg, gphys) + Du[:, :, None, :] * ch.Phi[None, :, :, None]
        out.append(np.einsum("eq,eqic,eqjc->eij", ch.W, gphys, Ddot))
    return np.concatenate(out)


def dense_jacobian(pr: Problem, u):
    """Assembled dF/du (N x N) from Eq. 3 element tangents; Dirichlet rows zero (A2)."""
    N = pr.n_dofs
    A = np.zeros((N, N))
    el = np.arange(pr.n_elems)
    Ke = element_tangent(pr, u, el)
    dofs = dof_map(pr, el)
    for e in range(len(el)):
        A[np.ix_(dofs[e], dofs[e])] += Ke[e]
    A[dirichlet_mask(pr), :] = 0.0
    return A
