"""1D rules of the oracle (test infrastructure only; see oracle/__init__.py).

* Gauss-Legendre points/weights on the reference interval [0,1] (reading A4),
  ``qorder`` = number of points per axis (reading A5).
* Gauss-Lobatto-Legendre (GLL) nodes of Q_k on [0,1] (reading A3): the two
  endpoints plus the roots of P_k'.
* Lagrange basis values and first derivatives by the product formula.

PAPER.md line 126-127 (operator B: "maps the solution field on the element
level to its gradients or values on the quadrature point level") needs exactly
these 1D ingredients; the paper fixes neither node set nor rule (A3, A5).
"""
from __future__ import annotations

import numpy as np
from numpy.polynomial import legendre as L


def gauss_legendre01(q: int):
    """q-point Gauss-Legendre rule mapped from [-1,1] to [0,1]: x=(1+t)/2, w/2."""
    t, w = L.leggauss(q)
    return (1.0 + t) / 2.0, w / 2.0


def gll_nodes01(k: int):
    """k+1 GLL nodes on [0,1] and their quadrature weights.

    Nodes: {-1, roots of P_k', +1} mapped by (1+t)/2. Weights on [-1,1] are
    2 / (k (k+1) P_k(t)^2); halved on [0,1].
    """
    if k < 1:
        raise ValueError("k >= 1")
    Pk = L.Legendre.basis(k)
    inner = np.sort(np.real(Pk.deriv().roots())) if k >= 2 else np.array([])
    t = np.concatenate([[-1.0], inner, [1.0]])
    w = 2.0 / (k * (k + 1) * Pk(t) ** 2)
    return (1.0 + t) / 2.0, w / 2.0


def lagrange_eval(nodes, x):
    """Values V[i,a] = l_a(x_i) and derivatives D[i,a] = l_a'(x_i).

    l_a(x) = prod_{m != a} (x - xi_m)/(xi_a - xi_m); the derivative is the
    product rule written out term by term.
    """
    nodes = np.asarray(nodes, dtype=np.float64)
    x = np.asarray(x, dtype=np.float64)
    n = len(nodes)
    V = np.ones((len(x), n))
    D = np.zeros((len(x), n))
    for a in range(n):
        for m in range(n):
            if m != a:
                V[:, a] *= (x - nodes[m]) / (nodes[a] - nodes[m])
        for m in range(n):
            if m == a:
                continue
            term = np.full(len(x), 1.0 / (nodes[a] - nodes[m]))
            for r in range(n):
                if r != a and r != m:
                    term *= (x - nodes[r]) / (nodes[a] - nodes[r])
            D[:, a] += term
    return V, D
