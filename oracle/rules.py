"""1D rules for the oracle (TEST INFRASTRUCTURE; see oracle/__init__.py).

* Gauss-Legendre quadrature with q points on the reference interval [0, 1], weights summing
  to 1 (reading R3 in DESIGN.md; SPEC.md:100-108 gives the same convention).
* Gauss-Lobatto-Legendre (GLL) nodes for degree p on [0, 1]: 0, 1 and the roots of
  P_p'(t) mapped by t -> (1 + t) / 2 (reading R2).
* Lagrange cardinal polynomials on the GLL nodes by the PRODUCT formula
  l_i(t) = prod_{j != i} (t - xi_j) / (xi_i - xi_j)
  and its derivative by the sum-of-products rule.  (The CUDA path's host code uses the
  barycentric form instead, so the two tables are computed independently.)

These are the 1D factors B_1D, D_1D of the tensor-product basis, PAPER.md:192-196 (Eq. 6,
"G_xi = D_1D (x) B_1D (x) B_1D").
"""

import numpy as np
from numpy.polynomial import legendre as L


def gauss_legendre(q):
    """Gauss-Legendre points and weights on [0, 1] (weights sum to 1)."""
    if q < 1:
        raise ValueError("q must be >= 1")
    t, w = L.leggauss(q)
    return (1.0 + t) / 2.0, w / 2.0


def gll_nodes(p):
    """GLL nodes on [0, 1] for degree p >= 1: endpoints plus mapped roots of P_p'.

    Roots come from numpy, are Newton-polished on P_p' and symmetrised
    (xi_{p-i} = 1 - xi_i) so that e.g. the p=6 midpoint is exactly 0.5.
    """
    if p < 1:
        raise ValueError("p must be >= 1")
    if p == 1:
        return np.array([0.0, 1.0])
    c = np.zeros(p + 1)
    c[p] = 1.0
    d1 = L.legder(c)          # P_p'
    d2 = L.legder(d1)         # P_p''
    r = np.sort(np.real(L.legroots(d1)))
    for _ in range(6):        # Newton polish on P_p'(t) = 0
        r = r - L.legval(r, d1) / L.legval(r, d2)
    t = np.concatenate(([-1.0], np.sort(r), [1.0]))
    t = 0.5 * (t - t[::-1])   # antisymmetric in t <=> symmetric about 1/2 on [0,1]
    x = (1.0 + t) / 2.0
    half = (p + 1) // 2
    x[p + 1 - half:] = 1.0 - x[:half][::-1]   # upper half mirrors the lower half
    if p % 2 == 0:
        x[p // 2] = 0.5
    x[0], x[-1] = 0.0, 1.0
    return x


def lagrange_values(nodes, t):
    """B[a, i] = l_i(t_a) by the product formula."""
    nodes = np.asarray(nodes, dtype=np.float64)
    t = np.atleast_1d(np.asarray(t, dtype=np.float64))
    n = nodes.size
    B = np.ones((t.size, n))
    for i in range(n):
        for j in range(n):
            if j != i:
                B[:, i] *= (t - nodes[j]) / (nodes[i] - nodes[j])
    return B


def lagrange_derivatives(nodes, t):
    """D[a, i] = l_i'(t_a) = sum_{m != i} 1/(xi_i - xi_m) prod_{j != i, m} (t - xi_j)/(xi_i - xi_j)."""
    nodes = np.asarray(nodes, dtype=np.float64)
    t = np.atleast_1d(np.asarray(t, dtype=np.float64))
    n = nodes.size
    D = np.zeros((t.size, n))
    for i in range(n):
        for m in range(n):
            if m == i:
                continue
            term = np.full(t.size, 1.0 / (nodes[i] - nodes[m]))
            for j in range(n):
                if j != i and j != m:
                    term *= (t - nodes[j]) / (nodes[i] - nodes[j])
            D[:, i] += term
    return D
