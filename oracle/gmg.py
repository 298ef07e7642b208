"""Oracle: geometric multigrid V-cycle (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

PAPER.md:197-218 (Sec. 3, Fig. 2): "A standard GMG V-cycle consists of three core components: a
smoother, inter-grid transfer operators, and a coarse-grid solver" -- "the inter-grid transfer
operators (restriction and prolongation) directly leverage the standard finite element
interpolation operators"; "a matrix-free Chebyshev polynomial smoother" on the fine levels; the
coarsest level solved "robustly" (AMG in the paper; a dense direct solve here, SPEC.md solvers
coarse_solve, reading R24).  Readings R22-R25 in DESIGN.md:

* hierarchy (R22): h-coarsening by 2 per axis, same p and q on every level; the coarse mesh's
  vertices are the fine vertices of even index; a coarse element's lambda, mu are the
  arithmetic means over its 8 children; the same Dirichlet faces on every level (SPEC).
* prolongation P (R23): finite element interpolation in reference coordinates.  Fine node
  with global index I_f along an axis lies in coarse element e = min(I_f // (2p), n_c - 1) at
  coarse reference coordinate t = (I_f - 2 p e) / (2 p) in fine-GLL spacing, i.e.
  xi_c = (s + xi_f(i)) / 2 with s the child index and xi_f the GLL node; u_f = sum_c
  l_c(xi_c) u_c (product-formula Lagrange, Eq. 6).  The 3D P is the Kronecker product of the
  three 1D operators (x fastest), applied per component.  Restriction R = P^T.
* V-cycle (R25): x = 0; pre-smooth (Chebyshev); r = b - A x with constrained fine entries
  zeroed; r_c = R r with constrained coarse entries zeroed; e_c = V(l-1, r_c); x += P e_c
  (constrained fine entries zeroed); post-smooth (same Chebyshev); coarsest: direct solve.
  Symmetric (pre = post, masked transfers Z_f P Z_c and its transpose), so usable as a CG
  preconditioner.
"""

import numpy as np

from .elasticity import Mesh, assemble_dense, constrained_mask
from .rules import gll_nodes, lagrange_values
from .solvers import chebyshev, diagonal, power_lambda_max


def coarsen(mesh):
    """The next coarser mesh (R22); None if some axis cannot be halved."""
    if mesh.nx % 2 or mesh.ny % 2 or mesh.nz % 2:
        return None
    V = mesh.vertices[::2, ::2, ::2]
    lam = np.asarray(mesh.lam)
    mu = np.asarray(mesh.mu)

    def avg(a):
        return 0.125 * sum(a[k::2, j::2, i::2] for k in (0, 1) for j in (0, 1) for i in (0, 1))

    return Mesh(V, mesh.p, mesh.q, avg(lam), avg(mu), mesh.dirichlet_faces)


def prolongation_1d(p, n_coarse):
    """(n_f x n_c) matrix of the 1D interpolation, n_f = 2 p n_coarse + 1 nodes (R23)."""
    xi = gll_nodes(p)
    Nc, Nf = n_coarse * p + 1, 2 * n_coarse * p + 1
    P = np.zeros((Nf, Nc))
    for If in range(Nf):
        e = min(If // (2 * p), n_coarse - 1)
        t = If - 2 * p * e                    # 0 .. 2p
        s, i = (0, t) if t < p else (1, t - p)
        xc = 0.5 * (s + xi[i])
        P[If, e * p:(e + 1) * p + 1] = lagrange_values(xi, np.array([xc]))[0]
    return P


def prolongation(fine, coarse):
    """Dense 3D P (3 N_f x 3 N_c), component-blocked: kron(Pz, kron(Py, Px)) per component."""
    p = fine.p
    Px = prolongation_1d(p, coarse.nx)
    Py = prolongation_1d(p, coarse.ny)
    Pz = prolongation_1d(p, coarse.nz)
    P1 = np.kron(Pz, np.kron(Py, Px))
    return np.kron(np.eye(3), P1)


class Level:
    def __init__(self, mesh, order, alpha, beta, power_iters, seed):
        self.mesh = mesh
        self.A = assemble_dense(mesh)
        self.d = diagonal(mesh)
        self.Z = constrained_mask(mesh)
        self.order, self.alpha, self.beta = order, alpha, beta
        from synth import splitmix_uniform
        v0 = splitmix_uniform(mesh.num_dofs, seed)
        self.lam = power_lambda_max(mesh, self.d, v0, power_iters, matvec=lambda v: self.A @ v)

    def smooth(self, b, x):
        return chebyshev(self.mesh, self.d, self.lam, self.order, self.alpha, self.beta, b, x,
                         matvec=lambda v: self.A @ v)


class GMG:
    """Levels finest first; dense operators (small meshes only: this is the oracle)."""

    def __init__(self, fine, levels, order=3, alpha=0.1, beta=1.1, power_iters=10, seed=1):
        meshes = [fine]
        while len(meshes) < levels:
            c = coarsen(meshes[-1])
            if c is None:
                raise ValueError("mesh cannot be coarsened that many times")
            meshes.append(c)
        self.levels = [Level(m, order, alpha, beta, power_iters, seed) for m in meshes]
        self.P = [prolongation(meshes[i], meshes[i + 1]) for i in range(len(meshes) - 1)]

    def vcycle(self, b, level=0):
        L = self.levels[level]
        if level == len(self.levels) - 1:
            return np.linalg.solve(L.A, b)
        x = L.smooth(b, np.zeros_like(b))
        r = b - L.A @ x
        r[L.Z] = 0.0                                  # constrained rows carry no residual down
        P = self.P[level]
        rc = P.T @ r
        rc[self.levels[level + 1].Z] = 0.0
        corr = P @ self.vcycle(rc, level + 1)
        corr[L.Z] = 0.0                               # (already 0: P maps face to face)
        return L.smooth(b, x + corr)
