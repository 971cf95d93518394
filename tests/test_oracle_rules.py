"""Pins T1-T3: the oracle's 1D rules and Lagrange basis.

The expected values come from closed forms (tests/golden/rules_1d.json) and
from mathematical properties computed here without the oracle's code path
(Bonnet's recurrence for Legendre polynomials, numpy.polynomial fits).
"""
import json
import math
import os

import numpy as np
import pytest
from numpy.polynomial import polynomial as Pl

import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "rules_1d.json")))


def _ev(s):
    return eval(s, {"sqrt": math.sqrt})


def _legendre_and_deriv(k, t):
    """Bonnet recurrence (independent of numpy.polynomial.legendre)."""
    t = np.asarray(t, float)
    p0, p1 = np.ones_like(t), t.copy()
    if k == 0:
        return p0, np.zeros_like(t)
    for n in range(1, k):
        p0, p1 = p1, ((2 * n + 1) * t * p1 - n * p0) / (n + 1)
    # (1 - t^2) P_k' = k (P_{k-1} - t P_k)
    with np.errstate(divide="ignore", invalid="ignore"):
        dp = k * (p0 - t * p1) / (1 - t * t)
    return p1, dp


@pytest.mark.parametrize("q", sorted(GOLD["gauss"], key=int))
def test_t1_gauss_closed_form(q):
    x, w = O.gauss_legendre01(int(q))
    t = np.array([_ev(s) for s in GOLD["gauss"][q]["t"]])
    wt = np.array([_ev(s) for s in GOLD["gauss"][q]["w"]])
    np.testing.assert_allclose(x, (1 + t) / 2, atol=1e-15)
    np.testing.assert_allclose(w, wt / 2, atol=1e-15)


@pytest.mark.parametrize("q", range(1, 10))
def test_t1_gauss_exactness(q):
    x, w = O.gauss_legendre01(q)
    for m in range(2 * q):
        assert abs(w @ x ** m - 1.0 / (m + 1)) < 2e-15
    # not exact one degree higher (the rule is exactly 2q-1)
    assert abs(w @ x ** (2 * q) - 1.0 / (2 * q + 1)) > 1e-13


def test_t1_app_b():
    g = GOLD["app_b_values_01"]
    x, w = O.gauss_legendre01(7)
    np.testing.assert_allclose(x, g["gauss7_x"], atol=1e-15)
    np.testing.assert_allclose(w[:4], g["gauss7_w_half"], atol=1e-15)
    # the tabulated points are the roots of P_7 (independent recurrence)
    P7, _ = _legendre_and_deriv(7, 2 * np.array(g["gauss7_x"]) - 1)
    assert np.max(np.abs(P7)) < 1e-13


@pytest.mark.parametrize("k", sorted(GOLD["gll"], key=int))
def test_t2_gll_closed_form(k):
    x, w = O.gll_nodes01(int(k))
    t = np.array([_ev(s) for s in GOLD["gll"][k]["t"]])
    wt = np.array([_ev(s) for s in GOLD["gll"][k]["w"]])
    np.testing.assert_allclose(x, (1 + t) / 2, atol=1e-15)
    np.testing.assert_allclose(w, wt / 2, atol=1e-15)


@pytest.mark.parametrize("k", range(1, 9))
def test_t2_gll_properties(k):
    x, w = O.gll_nodes01(k)
    assert x[0] == 0.0 and x[-1] == 1.0
    assert np.all(np.diff(x) > 0)
    assert abs(w[0] - 1.0 / (k * (k + 1))) < 1e-15
    # interior nodes are roots of P_k'
    if k >= 2:
        _, dP = _legendre_and_deriv(k, 2 * x[1:-1] - 1)
        assert np.max(np.abs(dP)) < 1e-11
    # GLL quadrature exact to degree 2k-1
    for m in range(2 * k):
        assert abs(w @ x ** m - 1.0 / (m + 1)) < 1e-14


def test_t2_app_b_gll6():
    x, _ = O.gll_nodes01(6)
    np.testing.assert_allclose(x, GOLD["app_b_values_01"]["gll6_x"], atol=1e-15)


@pytest.mark.parametrize("k", range(1, 8))
def test_t3_lagrange(k):
    nodes, _ = O.gll_nodes01(k)
    V, D = O.lagrange_eval(nodes, nodes)
    np.testing.assert_allclose(V, np.eye(k + 1), atol=1e-13)
    xs = np.linspace(-0.1, 1.1, 37)
    V, D = O.lagrange_eval(nodes, xs)
    np.testing.assert_allclose(V.sum(1), 1.0, atol=1e-13)
    np.testing.assert_allclose(D.sum(1), 0.0, atol=1e-11)
    # polynomial reproduction of values and derivatives for degree <= k
    for m in range(k + 1):
        np.testing.assert_allclose(V @ nodes ** m, xs ** m, atol=1e-12)
        np.testing.assert_allclose(D @ nodes ** m, m * xs ** max(m - 1, 0) if m else 0 * xs, atol=1e-10)
    # each cardinal function against an independent numpy polynomial fit
    for a in range(k + 1):
        c = Pl.polyfit(nodes, np.eye(k + 1)[a], k)
        np.testing.assert_allclose(V[:, a], Pl.polyval(xs, c), atol=1e-9)
        np.testing.assert_allclose(D[:, a], Pl.polyval(xs, Pl.polyder(c)), atol=1e-7)
