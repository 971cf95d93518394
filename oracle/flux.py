"""Pointwise operator D and its analytic derivatives (test infrastructure only).

D is "entirely local and is evaluated pointwise at every quadrature point"
(PAPER.md line 25); J_D = dD/du_q (Eq. 2). The oracle uses the
hand-coded ("HND", Table 1) derivatives below, never dual numbers.

Models (BASELINE.json configs; SPEC.md lines 304, 313, 330 for the forms):

* PLAPLACE (p-Laplacian, line 164):  D = k g,  k = (eps^2 + |g|^2)^((p-2)/2)
      dD/dg = k I + (p-2) s^((p-4)/2) g g^T ,  dD/du = 0
      p == 2: k = 1 and the second term is 0 (reading A12).
      eps == 0 and g == 0 (s == 0), p > 2: dD/dg = 0, the limit of both terms as
      g -> 0 (k ~ |g|^(p-2), (p-2) s^((p-4)/2) g g^T ~ |g|^(p-2)); written out so that
      0 * inf does not produce NaN (reading A20).
* NLDIFF (nonlinear diffusion):      D = (1+u^2) g
      dD/dg = (1+u^2) I ,  dD/du = 2 u g
* HEAT (design problem):             D = rho^3 (1+u^2) g
      dD/dg = rho^3 (1+u^2) I ,  dD/du = 2 rho^3 u g ,  dD/drho = 3 rho^2 (1+u^2) g

Arrays: U (...,), g (..., 3), rho broadcastable to U. Returns (..., 3) or (..., 3, 3).
"""
from __future__ import annotations

import numpy as np

PLAPLACE, NLDIFF, HEAT = 0, 1, 2


def _s(g, eps):
    return eps * eps + np.einsum("...i,...i->...", g, g)


def flux(model, U, g, p=2.0, eps=0.0, rho=None):
    if model == PLAPLACE:
        if p == 2.0:
            return g.copy()
        k = _s(g, eps) ** ((p - 2.0) / 2.0)
        return k[..., None] * g
    if model == NLDIFF:
        return (1.0 + U * U)[..., None] * g
    if model == HEAT:
        return (rho ** 3 * (1.0 + U * U))[..., None] * g
    raise ValueError(model)


def flux_dg(model, U, g, p=2.0, eps=0.0, rho=None):
    """dD/dg as (..., 3, 3)."""
    eye = np.eye(3)
    if model == PLAPLACE:
        if p == 2.0:
            return np.broadcast_to(eye, g.shape + (3,)).copy()
        s = _s(g, eps)
        k = s ** ((p - 2.0) / 2.0)
        pos = s > 0.0
        c = np.where(pos, (p - 2.0) * np.where(pos, s, 1.0) ** ((p - 4.0) / 2.0), 0.0)   # A20 at s == 0
        return k[..., None, None] * eye + c[..., None, None] * g[..., :, None] * g[..., None, :]
    if model == NLDIFF:
        return (1.0 + U * U)[..., None, None] * eye
    if model == HEAT:
        return (rho ** 3 * (1.0 + U * U))[..., None, None] * eye
    raise ValueError(model)


def flux_du(model, U, g, p=2.0, eps=0.0, rho=None):
    """dD/du as (..., 3)."""
    if model == PLAPLACE:
        return np.zeros_like(g)
    if model == NLDIFF:
        return (2.0 * U)[..., None] * g
    if model == HEAT:
        return (2.0 * rho ** 3 * U)[..., None] * g
    raise ValueError(model)


def flux_drho(model, U, g, p=2.0, eps=0.0, rho=None):
    """dD/drho as (..., 3); only the HEAT model depends on rho."""
    if model == HEAT:
        return (3.0 * rho ** 2 * (1.0 + U * U))[..., None] * g
    return np.zeros_like(g)
