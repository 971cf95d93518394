"""Jacobian-free Newton with unpreconditioned CG (test infrastructure only).

PAPER.md line 164 / 211 ("matrix-free non-linear solvers"), BASELINE.json
configs[3], reading A15:

    u = u0
    repeat newton_steps times:
        F = F(u);  record ||F||
        CG on J(u) delta = -F from delta = 0, exactly cg_iters iterations,
           no preconditioner, no convergence test; p^T J p <= 0 is an error
        u = u + delta
    record ||F(u)||

Uses only ``residual`` and ``jvp`` of this oracle. Beyond roundoff growth the
free-running trajectory is "parity unpinned" (T17): the tests compare it state-
synchronised (each Newton iterate and CG direction fed to both sides).
"""
from __future__ import annotations

import numpy as np

from .fem import residual, jvp, element_tangent, dof_map, dirichlet_mask


def cg_fixed(apply, b, iters, diag=None):
    """Plain CG (Hestenes-Stiefel) from x = 0 for a fixed number of iterations;
    with ``diag`` the Jacobi-preconditioned CG (z = r / diag)."""
    x = np.zeros_like(b)
    r = b.copy()
    z = r / diag if diag is not None else r.copy()
    p = z.copy()
    rz = float(r @ z)
    dirs = []
    for _ in range(iters):
        Ap = apply(p)
        pAp = float(p @ Ap)
        if not pAp > 0.0:
            raise FloatingPointError("CG breakdown: p^T A p <= 0")
        alpha = rz / pAp
        dirs.append(p.copy())
        x += alpha * p
        r -= alpha * Ap
        z = r / diag if diag is not None else r
        rz_new = float(r @ z)
        p = z + (rz_new / rz) * p
        rz = rz_new
    return x, dirs


def jacobi_diag(pr, u):
    """Diagonal of J(u) (Eq. 3 element tangents, diagonal entries scattered with
    numpy.bincount) on free rows, 1 on Dirichlet rows (J's rows there are zero)."""
    el = np.arange(pr.n_elems)
    Ke = element_tangent(pr, u, el)
    dofs = dof_map(pr, el)
    d = np.bincount(dofs.ravel(), weights=np.einsum("eii->ei", Ke).ravel(), minlength=pr.n_dofs)
    d[dirichlet_mask(pr)] = 1.0
    return d


def newton_cg(pr, u0, newton_steps=5, cg_iters=20, record=False, jacobi=False):
    u = np.array(u0, dtype=np.float64)
    norms = []
    iterates = []
    directions = []
    for _ in range(newton_steps):
        F = residual(pr, u)
        norms.append(float(np.linalg.norm(F)))
        iterates.append(u.copy())
        delta, dirs = cg_fixed(lambda x: jvp(pr, u, x), -F, cg_iters, jacobi_diag(pr, u) if jacobi else None)
        directions.append(dirs)
        u = u + delta
    norms.append(float(np.linalg.norm(residual(pr, u))))
    if record:
        return u, norms, iterates, directions
    return u, norms


def bicgstab_fixed(apply, b, iters):
    """Unpreconditioned BiCGStab (van der Vorst 1992) from x = 0, shadow residual
    rhat = b, for a fixed number of iterations; a converged state (r = 0) freezes.
    Returns x and the recursive residual norms (before the first and after each
    iteration). Reference for feod_adjoint_solve's iteration."""
    x = np.zeros_like(b)
    r = b.copy()
    rhat = b.copy()
    p = np.zeros_like(b)
    v = np.zeros_like(b)
    rho_old = alpha = omega = 0.0
    hist = [float(np.linalg.norm(r))]
    for it in range(iters):
        rho = float(rhat @ r)
        if it == 0:
            p = r.copy()
        else:
            beta = 0.0 if (rho_old == 0.0 or omega == 0.0) else (rho / rho_old) * (alpha / omega)
            p = r + beta * (p - omega * v)
        v = apply(p)
        rv = float(rhat @ v)
        alpha = rho / rv if rv != 0.0 else 0.0
        s = r - alpha * v
        t = apply(s)
        tt = float(t @ t)
        omega = float(t @ s) / tt if tt > 0.0 else 0.0
        x = x + alpha * p + omega * s
        r = s - omega * t
        rho_old = rho
        hist.append(float(np.linalg.norm(r)))
    return x, hist
