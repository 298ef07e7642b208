"""Pins for the oracle's 1D rules and basis tables (closed forms, exactness, sympy roots).

Citations: quadrature/basis conventions SPEC.md:100-130; tensor-product basis PAPER.md:192-196.
"""

import json
import math
import os

import numpy as np
import pytest
import sympy as sp

from oracle import rules

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_gauss_legendre_closed_forms():
    g, w = rules.gauss_legendre(1)
    assert np.allclose(g, [0.5], atol=0, rtol=0) and np.allclose(w, [1.0], atol=0, rtol=0)
    g, w = rules.gauss_legendre(2)
    s = math.sqrt(3.0) / 6.0
    assert np.allclose(g, [0.5 - s, 0.5 + s], atol=1e-16)
    assert np.allclose(w, [0.5, 0.5], atol=1e-16)
    with pytest.raises(ValueError):
        rules.gauss_legendre(0)


@pytest.mark.parametrize("q", range(1, 12))
def test_gauss_legendre_exactness(q):
    g, w = rules.gauss_legendre(q)
    assert abs(w.sum() - 1.0) < 1e-14
    assert np.all(np.diff(g) > 0) and np.all(w > 0)
    for k in range(2 * q):              # exact for degree <= 2q-1
        assert abs(np.dot(w, g ** k) - 1.0 / (k + 1)) < 1e-14
    # and NOT exact at degree 2q (the rule really has q points); the defect shrinks fast
    if q <= 6:
        assert abs(np.dot(w, g ** (2 * q)) - 1.0 / (2 * q + 1)) > 1e-10


def test_gll_closed_forms():
    assert np.array_equal(rules.gll_nodes(1), [0.0, 1.0])
    assert np.allclose(rules.gll_nodes(2), [0.0, 0.5, 1.0], atol=0)
    r5 = 1.0 / math.sqrt(5.0)
    assert np.allclose(rules.gll_nodes(3), [0, (1 - r5) / 2, (1 + r5) / 2, 1], atol=2e-16)
    r = math.sqrt(3.0 / 7.0)
    assert np.allclose(rules.gll_nodes(4), [0, (1 - r) / 2, 0.5, (1 + r) / 2, 1], atol=2e-16)
    with pytest.raises(ValueError):
        rules.gll_nodes(0)


@pytest.mark.parametrize("p", range(2, 9))
def test_gll_against_sympy_roots(p):
    """Interior GLL nodes = roots of P_p' (independent: sympy's Legendre + 30-digit nroots)."""
    t = sp.Symbol("t")
    roots = sorted(float((1 + r) / 2) for r in sp.Poly(sp.diff(sp.legendre(p, t), t), t).nroots(n=30))
    x = rules.gll_nodes(p)
    assert np.allclose(x[1:-1], roots, atol=2e-16, rtol=0)
    assert np.allclose(x, 1.0 - x[::-1], atol=1.2e-16, rtol=0)  # symmetry to 1 ulp
    if p % 2 == 0:
        assert x[p // 2] == 0.5


def test_golden_1d_values():
    """SURVEY Appendix B.3 values (derived independently; re-checked here)."""
    with open(os.path.join(GOLDEN, "rules_1d.json")) as f:
        gold = json.load(f)
    for p, vals in gold["gll_interior_lower_half"].items():
        x = rules.gll_nodes(int(p))
        assert np.allclose(x[1:1 + len(vals)], vals, atol=1e-15)
    g, w = rules.gauss_legendre(10)
    assert abs(g[0] - gold["gl_q10_first"]["point"]) < 1e-15
    assert abs(w[0] - gold["gl_q10_first"]["weight"]) < 1e-15


@pytest.mark.parametrize("p,q", [(1, 1), (1, 3), (2, 4), (3, 5), (4, 5), (5, 7), (6, 8), (7, 9), (8, 10), (8, 9)])
def test_basis_tables(p, q):
    nodes = rules.gll_nodes(p)
    g, _ = rules.gauss_legendre(q)
    B = rules.lagrange_values(nodes, g)
    D = rules.lagrange_derivatives(nodes, g)
    assert B.shape == (q, p + 1) and D.shape == (q, p + 1)
    assert np.allclose(B.sum(axis=1), 1.0, atol=1e-13)          # partition of unity
    assert np.allclose(D.sum(axis=1), 0.0, atol=1e-12)          # derivative of a constant
    assert np.allclose(rules.lagrange_values(nodes, nodes), np.eye(p + 1), atol=1e-14)  # Lagrange property
    for k in range(p + 1):                                       # exact on degree <= p
        assert np.allclose(B @ nodes ** k, g ** k, atol=1e-13)
        dk = k * g ** (k - 1) if k > 0 else np.zeros_like(g)
        assert np.allclose(D @ nodes ** k, dk, atol=1e-11)
    # symmetry of the symmetric node/point sets: B[q-1-a, n-1-i] = B[a, i], D antisymmetric
    assert np.allclose(B[::-1, ::-1], B, atol=1e-14)
    assert np.allclose(D[::-1, ::-1], -D, atol=1e-12)


def test_basis_p1_q1_example():
    """p=1, q=1 -> B = [[0.5, 0.5]], D = [[-1, 1]]."""
    nodes = rules.gll_nodes(1)
    g, _ = rules.gauss_legendre(1)
    assert np.allclose(rules.lagrange_values(nodes, g), [[0.5, 0.5]], atol=0)
    assert np.allclose(rules.lagrange_derivatives(nodes, g), [[-1.0, 1.0]], atol=0)


def test_derivative_vs_finite_differences():
    """D columns agree with centred differences of the cardinal functions."""
    nodes = rules.gll_nodes(4)
    g, _ = rules.gauss_legendre(5)
    h = 1e-5
    fd = (rules.lagrange_values(nodes, g + h) - rules.lagrange_values(nodes, g - h)) / (2 * h)
    assert np.allclose(rules.lagrange_derivatives(nodes, g), fd, atol=1e-6)
