"""Oracle: matrix-free diagonal, power-iteration spectral estimate, Chebyshev smoother, PCG.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py for who may import this).  Plain numpy
FP64, no code shared with the CUDA path.  These are the consumers of the apply in the paper's
solver:

* diagonal(mesh): diag of A (Eq. 5) written out from Eqs. 3-4 with i = j, I = J:
      A[(c,I),(c,I)] = sum_e sum_qp W [(lambda + mu) (d_c phi_I)^2 + mu |grad phi_I|^2],
  Dirichlet rows -> 1 (the operator y = Z A Z x + (I - Z) x, reading R9).  SPEC.md
  "assemble_diagonal" (needed by Jacobi and Chebyshev).
* power_lambda_max(mesh, d, v0, iters): "an estimate of the operator's spectral radius ...
  a few Lanczos or power iterations" (Sec. 3.1); SPEC.md solvers
  power_iteration_lambda_max: power iteration on D^{-1} A, times the 1.1 safety factor
  (reading R19 in DESIGN.md: v <- v/|v|; w = D^{-1} A v; lambda = v.w; v <- w/|w|).
* chebyshev(mesh, d, lam_max, order, alpha, beta, b, x): "applying a polynomial of the
  operator A to the residual": x <- x + p_k(D^{-1}A) D^{-1} (b - A x), p_k the
  degree-k Chebyshev polynomial for the interval [alpha lam_max, beta lam_max] (SPEC.md
  solvers chebyshev_smooth; defaults k = 3, alpha = 0.1, beta = 1.1, reading R20), by the
  classical three-term Chebyshev iteration (Saad, Iterative Methods, Alg. 12.1).
* pcg(mesh, b, precond, rtol, maxit): preconditioned conjugate gradients ("CG algorithm being
  the method of choice"), zero initial guess, stopped on the preconditioned
  residual sqrt(r.z) relative to its initial value (SPEC.md solvers cg_solve).

Pins (tests/test_oracle_solvers.py): the diagonal against diag of the assembled matrix and of
the independent Kronecker assembly; the Chebyshev error polynomial against the closed form
T_k((theta - lambda)/delta) / T_k(theta/delta) on every eigenvector of a dense D^{-1/2}AD^{-1/2};
power iteration against the SPEC examples and dense eigenvalues; PCG against a dense solve.
"""

import numpy as np

from .elasticity import (
    apply,
    constrained_mask,
    element_geometry,
    element_nodes,
    element_vertices,
    reference_tables,
    _elements,
)

SAFETY = 1.1


def diagonal(mesh):
    """diag(Z A Z + (I - Z)) by the definition above (element loop, no sum factorisation)."""
    N = mesh.num_nodes
    Gref, w3, g = reference_tables(mesh.p, mesh.q)
    d = np.zeros(3 * N)
    for ex, ey, ez in _elements(mesh):
        J, detJ, W = element_geometry(element_vertices(mesh, ex, ey, ez), g, w3)
        A = np.linalg.inv(J)
        Phi = np.einsum("klq,qkm->mlq", Gref, A)            # Phi[m][l, qp] = d_m phi_l
        nodes = element_nodes(mesh, ex, ey, ez)
        if mesh.C6 is not None:   # Eq. 2: sum_qp W sum_kl d_k phi C_ckcl d_l phi
            from .elasticity import VOIGT
            C6 = mesh.C6[ez, ey, ex]
            PP = np.einsum("kiq,liq,q->kli", Phi, Phi, W)               # (3, 3, n^3)
            for c in range(3):
                Cc = C6[VOIGT[c][:, None], VOIGT[c][None, :]]           # Cc[k, l] = C_ckcl
                np.add.at(d, c * N + nodes, np.einsum("kl,kli->i", Cc, PP))
            continue
        lam, mu = mesh.lam[ez, ey, ex], mesh.mu[ez, ey, ex]
        sq = np.einsum("mlq,q->ml", Phi ** 2, W)             # sum_qp W (d_m phi_l)^2
        tot = sq.sum(axis=0)
        for c in range(3):
            np.add.at(d, c * N + nodes, (lam + mu) * sq[c] + mu * tot)
    d[constrained_mask(mesh)] = 1.0
    return d


def power_lambda_max(mesh, d, v0, iters, matvec=None):
    """1.1 x the power-iteration estimate of the largest eigenvalue of D^{-1} A."""
    A = matvec or (lambda v: apply(mesh, v))
    v = np.asarray(v0, dtype=np.float64) / np.linalg.norm(v0)
    lam = 0.0
    for _ in range(iters):
        w = A(v) / d
        lam = float(v @ w)
        v = w / np.linalg.norm(w)
    return SAFETY * lam


def chebyshev(mesh, d, lam_max, order, alpha, beta, b, x, matvec=None):
    """One Chebyshev smoothing pass: returns x + p_k(D^{-1}A) D^{-1} (b - A x)."""
    A = matvec or (lambda v: apply(mesh, v))
    lo, hi = alpha * lam_max, beta * lam_max
    theta, delta = 0.5 * (hi + lo), 0.5 * (hi - lo)
    x = np.array(x, dtype=np.float64, copy=True)
    r = (b - A(x)) / d
    dvec = r / theta
    if order > 1:
        sigma = theta / delta
        rho = 1.0 / sigma
    for k in range(1, order + 1):
        x += dvec
        if k == order:
            break
        r = r - A(dvec) / d
        rho_new = 1.0 / (2.0 * sigma - rho)
        dvec = rho_new * rho * dvec + (2.0 * rho_new / delta) * r
        rho = rho_new
    return x


def pcg(mesh, b, precond, rtol, maxit, matvec=None):
    """PCG from x0 = 0.  precond: callable r -> z (or None for none).

    Returns (x, iterations, history) with history[i] = sqrt(r_i . z_i) / sqrt(r_0 . z_0).
    Stops when history <= rtol or after maxit iterations.
    """
    A = matvec or (lambda v: apply(mesh, v))
    M = precond or (lambda r: r.copy())
    b = np.asarray(b, dtype=np.float64)
    x = np.zeros_like(b)
    r = b.copy()
    z = M(r)
    rz = float(r @ z)
    hist = [1.0]
    if rz == 0.0:
        return x, 0, hist
    rz0 = rz
    p = z.copy()
    it = 0
    while it < maxit:
        t = A(p)
        pt = float(p @ t)
        if pt <= 0.0:
            raise ArithmeticError("PCG: operator not positive definite")
        alpha = rz / pt
        x += alpha * p
        r -= alpha * t
        z = M(r)
        rz_new = float(r @ z)
        it += 1
        hist.append(np.sqrt(max(rz_new, 0.0) / rz0))
        if hist[-1] <= rtol:
            break
        beta = rz_new / rz
        p = z + beta * p
        rz = rz_new
    return x, it, hist
