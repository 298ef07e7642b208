"""Pins for the oracle's solver pieces (no GPU): diagonal, power iteration, Chebyshev, PCG.

* diagonal == diag of the assembled matrix and of the independent Kronecker assembly
  (exactly integrated 1D matrices, no quadrature)                        SPEC assemble_diagonal
* Chebyshev error polynomial == closed form T_k((theta-lam)/delta)/T_k(theta/delta) on every
  eigenvector of the dense D^{-1/2} A D^{-1/2} (cosh/cos form of T_k, independent of the
  three-term recurrence)                                           PAPER.md:209, SPEC chebyshev_smooth
* power iteration: SPEC examples (identity -> 1.1, diag(1,2,3) -> 3.3) and a dense eigensolve
* PCG == dense solve; zero rhs -> 0 iterations; Chebyshev-preconditioned needs fewer
  iterations than Jacobi                                                    SPEC cg_solve
"""

import numpy as np
import pytest

import oracle
import synth
from tests.test_oracle_operator import kron_operator, mesh_of


def small(p, dims=(2, 2, 2), faces=0, seed=3, perturb=True):
    return synth.make_problem("t", *dims, p, p + 2, perturb=perturb, lognormal_material=perturb,
                              faces=faces, seed=seed)


@pytest.mark.parametrize("p", [1, 2, 3, 4])
@pytest.mark.parametrize("faces", [0, 1 | 32])
def test_diagonal_equals_assembled(p, faces):
    m = mesh_of(small(p, faces=faces, seed=10 + p))
    d = oracle.diagonal(m)
    A = oracle.assemble_dense(m)
    assert np.abs(d - np.diag(A)).max() <= 1e-13 * np.abs(d).max()
    assert (d > 0).all()


@pytest.mark.parametrize("p,dims,lengths", [(1, (2, 3, 2), (1.0, 1.5, 0.7)), (3, (2, 1, 2), (0.6, 1.0, 1.3)),
                                            (4, (1, 1, 1), (1.0, 0.8, 1.2))])
def test_diagonal_equals_kronecker(p, dims, lengths):
    lam, mu = 1.3, 0.7
    P = synth.make_problem("t", *dims, p, p + 1, lengths=lengths, lam=lam, mu=mu, seed=1)
    d = oracle.diagonal(mesh_of(P))
    Ak = kron_operator(*dims, *lengths, p, lam, mu)
    assert np.abs(d - np.diag(Ak)).max() <= 1e-12 * np.abs(d).max()


def cheb_T(k, t):
    t = np.asarray(t, dtype=np.float64)
    out = np.empty_like(t)
    big = np.abs(t) >= 1
    out[big] = np.sign(t[big]) ** k * np.cosh(k * np.arccosh(np.abs(t[big])))
    out[~big] = np.cos(k * np.arccos(t[~big]))
    return out


@pytest.mark.parametrize("order", [1, 2, 3, 5])
@pytest.mark.parametrize("faces", [0, 1])
def test_chebyshev_error_polynomial_closed_form(order, faces):
    m = mesh_of(small(2, faces=faces, seed=4))
    A = oracle.assemble_dense(m)
    d = np.diag(A).copy()
    mv = lambda v: A @ v
    s = 1.0 / np.sqrt(d)
    ev, U = np.linalg.eigh(s[:, None] * A * s[None, :])      # D^{-1/2} A D^{-1/2} = U diag(ev) U^T
    lam_max = 1.1 * ev.max()
    alpha, beta = 0.1, 1.1
    rng = np.random.default_rng(0)
    x_star = rng.standard_normal(A.shape[0])
    b = A @ x_star
    x0 = rng.standard_normal(A.shape[0])
    x1 = oracle.chebyshev(m, d, lam_max, order, alpha, beta, b, x0, matvec=mv)
    # error e = x - x*: in the D^{1/2}-scaled eigenbasis each component is multiplied by
    # T_k((theta - lam)/delta) / T_k(theta/delta)
    lo, hi = alpha * lam_max, beta * lam_max
    theta, delta = (hi + lo) / 2, (hi - lo) / 2
    fac = cheb_T(order, (theta - ev) / delta) / cheb_T(order, np.array([theta / delta]))[0]
    c0 = U.T @ ((x0 - x_star) / s)
    c1 = U.T @ ((x1 - x_star) / s)
    assert np.abs(c1 - fac * c0).max() <= 1e-10 * np.abs(c0).max()


def test_chebyshev_fixed_point_and_linearity():
    m = mesh_of(small(2, seed=5))
    A = oracle.assemble_dense(m)
    d = np.diag(A).copy()
    mv = lambda v: A @ v
    rng = np.random.default_rng(1)
    x = rng.standard_normal(A.shape[0])
    assert np.allclose(oracle.chebyshev(m, d, 3.0, 3, 0.1, 1.1, A @ x, x, matvec=mv), x, rtol=0, atol=1e-13 * np.abs(x).max())
    x1, x2, b1, b2 = (rng.standard_normal(A.shape[0]) for _ in range(4))
    s = oracle.chebyshev(m, d, 3.0, 3, 0.1, 1.1, b1 + b2, x1 + x2, matvec=mv)
    t = oracle.chebyshev(m, d, 3.0, 3, 0.1, 1.1, b1, x1, matvec=mv) + oracle.chebyshev(m, d, 3.0, 3, 0.1, 1.1, b2, x2, matvec=mv)
    assert np.abs(s - t).max() <= 1e-12 * np.abs(s).max()


def test_chebyshev_one_by_one_exact():
    # SPEC: 1x1 system A = [2], D = [2], exact bounds -> one step solves exactly (order 1)
    x = oracle.chebyshev(None, np.array([2.0]), 1.0, 1, 1.0, 1.0, np.array([3.0]), np.array([0.0]),
                         matvec=lambda v: 2.0 * v)
    assert x[0] == 1.5


def test_power_iteration_spec_examples():
    n = 7
    v0 = synth.splitmix_uniform(n, 9)
    lam = oracle.power_lambda_max(None, np.ones(n), v0, 3, matvec=lambda v: v)
    assert abs(lam - 1.1) <= 1e-10
    lam = oracle.power_lambda_max(None, np.ones(3), synth.splitmix_uniform(3, 1), 50,
                                  matvec=lambda v: np.array([1.0, 2.0, 3.0]) * v)
    assert abs(lam - 3.3) <= 0.033


@pytest.mark.parametrize("p,faces", [(1, 1), (2, 0), (3, 1 | 2)])
def test_power_iteration_bounds_dense(p, faces):
    """Estimate within [1.0, 1.21] x the true lambda_max of D^{-1} A (SPEC example)."""
    m = mesh_of(small(p, faces=faces, seed=6))
    A = oracle.assemble_dense(m)
    d = oracle.diagonal(m)
    s = 1.0 / np.sqrt(d)
    true = np.linalg.eigvalsh(s[:, None] * A * s[None, :]).max()
    lam = oracle.power_lambda_max(m, d, synth.splitmix_uniform(m.num_dofs, 2), 30)
    assert 1.0 * true <= lam <= 1.21 * true


def test_splitmix_reference_values():
    """splitmix64 reference outputs (seed 0: the published first values of the generator)."""
    with np.errstate(over="ignore"):
        u = synth.splitmix_uniform(2, 0)
    z0 = 0xE220A8397B1DCDAF   # splitmix64 stream from state 0, first output
    assert u[0] == 2.0 * (z0 >> 11) * 2.0 ** -53 - 1.0
    assert np.all((u >= -1) & (u < 1))


@pytest.mark.parametrize("prec", ["none", "jacobi", "cheb"])
def test_pcg_matches_dense_solve(prec):
    m = mesh_of(small(2, dims=(2, 2, 3), faces=1, seed=7))
    A = oracle.assemble_dense(m)
    d = oracle.diagonal(m)
    b = synth.splitmix_uniform(m.num_dofs, 3)
    lam = oracle.power_lambda_max(m, d, synth.splitmix_uniform(m.num_dofs, 4), 10)
    M = {"none": None, "jacobi": lambda r: r / d,
         "cheb": lambda r: oracle.chebyshev(m, d, lam, 3, 0.1, 1.1, r, np.zeros_like(r))}[prec]
    x, it, hist = oracle.pcg(m, b, M, 1e-11, 2000)
    xs = np.linalg.solve(A, b)
    assert hist[-1] <= 1e-11
    assert np.linalg.norm(x - xs) <= 1e-8 * np.linalg.norm(xs)
    assert it > 0


def test_pcg_zero_rhs_and_preconditioner_ordering():
    m = mesh_of(small(2, dims=(3, 2, 2), faces=1, seed=8))
    d = oracle.diagonal(m)
    x, it, _ = oracle.pcg(m, np.zeros(m.num_dofs), lambda r: r / d, 1e-8, 100)
    assert it == 0 and not x.any()
    b = synth.splitmix_uniform(m.num_dofs, 5)
    lam = oracle.power_lambda_max(m, d, synth.splitmix_uniform(m.num_dofs, 6), 10)
    _, it_j, _ = oracle.pcg(m, b, lambda r: r / d, 1e-8, 2000)
    _, it_c, _ = oracle.pcg(m, b, lambda r: oracle.chebyshev(m, d, lam, 3, 0.1, 1.1, r, np.zeros_like(r)), 1e-8, 2000)
    assert it_c < it_j
