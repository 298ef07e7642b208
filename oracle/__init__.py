"""Plain, slow CPU oracle for the elasticity operator y = A x (TEST INFRASTRUCTURE ONLY).

This package is the independent definition the CUDA path is checked against.  It shares
no code with ``paper_2601_08374_b200`` (the product) and neither imports the other; the
only module both sides use is ``synth`` (seeded input generators, no method arithmetic).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import or execute anything under ``oracle/``.  The product
path never routes through it.

What it computes (Eq. 5): A_ij = a(phi_i, phi_j) with the bilinear form
a(u, v) = int sigma(u) : grad v  (Eq. 4) and isotropic Hooke's law
sigma = lambda (div u) I + 2 mu eps(u)  (Eq. 3), discretised with
tensor-product Q_p Lagrange elements (Eq. 6) on trilinear hexahedra.
Every element matrix is formed explicitly by naive quadrature ("explicitly calculating
each local matrix") and applied element by element.  No sum factorisation,
no Voigt packing, no stored quadrature data.

Readings of the paper where it is silent are listed in DESIGN.md section 3 (node placement
GLL, Gauss-Legendre quadrature with q points, reference cube [0,1]^3, component-blocked
vectors, lexicographic x-fastest numbering, Dirichlet rows/cols replaced by identity).

Pins (tests/test_oracle_*.py, ``-m "not gpu"``): closed-form 1D rules, exact Q1 element
matrix (sympy exact integration), exact rational invariants of config 1, rigid-body null
space, symmetry, PSD, patch-test energy, interior equilibrium, BC identity rows.  Every
function here is pinned; none is "parity unpinned".
"""

from .rules import gauss_legendre, gll_nodes, lagrange_values, lagrange_derivatives  # noqa: F401
from .elasticity import (  # noqa: F401
    Mesh,
    element_stiffness,
    apply,
    apply_elements,
    apply_rows,
    assemble_dense,
    constrained_mask,
    node_coordinates,
)
from .solvers import diagonal, power_lambda_max, chebyshev, pcg  # noqa: F401
from . import gmg  # noqa: F401
