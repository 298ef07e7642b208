"""Pins for the oracle operator against what the paper's setting fixes (no GPU).

* exact Q1 element matrix by symbolic integration (sympy)                      Eqs. 3-5
* exact global operator on affine boxes by an independent Kronecker assembly of
  exactly-integrated 1D matrices (no quadrature, no geometry code)           Eqs. 3-6
* exact rational invariants of config 1 (re-derived here in Fractions)
* rigid-body null space, symmetry, PSD, nullity 6 (PAPER.md:156 symmetric form)
* patch test x^T A x = Vol (lam tr(eps)^2 + 2 mu eps:eps) (north_star)
* interior equilibrium for affine fields, BC identity rows
"""

import json
import os
from fractions import Fraction

import numpy as np
import pytest
import sympy as sp

import oracle
import synth
from oracle import elasticity as E

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def mesh_of(P):
    lam, mu = P.material_arrays()
    return oracle.Mesh(P.vertex_array(), P.p, P.q, lam, mu, P.dirichlet_faces)


# ---------------------------------------------------------------------------------------
# Independent exact constructions
# ---------------------------------------------------------------------------------------

def q1_element_matrix_sympy(lam, mu):
    """Unit-cube Q1 element stiffness by exact symbolic integration of Eqs. 3-5."""
    x, y, z = sp.symbols("x y z")
    X = (x, y, z)
    phis = []
    for k in range(2):
        for j in range(2):
            for i in range(2):
                phis.append((x if i else 1 - x) * (y if j else 1 - y) * (z if k else 1 - z))
    grads = [[sp.diff(f, v) for v in X] for f in phis]
    n = 8
    K = sp.zeros(3 * n, 3 * n)
    integ = {}

    def I(a, b, A, B):
        key = (a, b, A, B)
        if key not in integ:
            # exact: int_0^1 x^i y^j z^k = 1 / ((i+1)(j+1)(k+1)), term by term
            poly = sp.Poly(sp.expand(grads[a][A] * grads[b][B]), x, y, z)
            integ[key] = sum(c / ((i + 1) * (j + 1) * (k + 1)) for (i, j, k), c in poly.terms())
        return integ[key]

    for i in range(3):
        for a in range(n):
            for j in range(3):
                for b in range(n):
                    v = lam * I(a, b, i, j) + mu * I(a, b, j, i)
                    if i == j:
                        v += mu * sum(I(a, b, m, m) for m in range(3))
                    K[i * n + a, j * n + b] = v
    return K


def lagrange_polys(nodes):
    """Cardinal polynomials as coefficient objects (exact integration instead of quadrature)."""
    P = np.polynomial.Polynomial
    out = []
    for i, xi in enumerate(nodes):
        others = [xj for j, xj in enumerate(nodes) if j != i]
        poly = P.fromroots(others)
        out.append(poly / poly(xi))
    return out


def one_d_global(nodes, ne, h):
    """Global 1D matrices on ne elements of size h: M = int phi phi, K = int phi' phi', C = int phi' phi."""
    p = len(nodes) - 1
    L = lagrange_polys(nodes)
    dL = [l.deriv() for l in L]

    def integ(f):
        F = f.integ()
        return F(1.0) - F(0.0)

    m = np.array([[integ(L[a] * L[b]) for b in range(p + 1)] for a in range(p + 1)])
    k = np.array([[integ(dL[a] * dL[b]) for b in range(p + 1)] for a in range(p + 1)])
    c = np.array([[integ(dL[a] * L[b]) for b in range(p + 1)] for a in range(p + 1)])
    N = ne * p + 1
    M, K, C = np.zeros((N, N)), np.zeros((N, N)), np.zeros((N, N))
    for e in range(ne):
        s = slice(e * p, e * p + p + 1)
        M[s, s] += h * m
        K[s, s] += k / h
        C[s, s] += c
    return M, K, C


def kron_operator(nx, ny, nz, lx, ly, lz, p, lam, mu, frac_nodes=None):
    """Global A for an axis-aligned uniform box with constant material, by Kronecker products.

    S_ab[(I),(J)] = int d_a phi_I d_b phi_J factorises into 1D integrals; with x fastest the
    3D matrix is kron(z, kron(y, x)).  A block (c,d) = lam S_cd + mu S_dc + mu delta_cd tr S.
    """
    from oracle.rules import gll_nodes
    nodes = gll_nodes(p)
    Mx, Kx, Cx = one_d_global(nodes, nx, lx / nx)
    My, Ky, Cy = one_d_global(nodes, ny, ly / ny)
    Mz, Kz, Cz = one_d_global(nodes, nz, lz / nz)
    k3 = lambda a, b, c: np.kron(c, np.kron(b, a))
    # d/dx uses (K or C) in x, etc.  Entry S_ab[I,J]: derivative a on I, b on J.
    # 1D factor for (deriv on I?, deriv on J?): (0,0)->M, (1,1)->K, (1,0)->C, (0,1)->C^T
    def f1(M, K, C, dI, dJ):
        return {(0, 0): M, (1, 1): K, (1, 0): C, (0, 1): C.T}[(dI, dJ)]
    mats = [(Mx, Kx, Cx), (My, Ky, Cy), (Mz, Kz, Cz)]
    S = [[None] * 3 for _ in range(3)]
    for a in range(3):
        for b in range(3):
            fac = [f1(*mats[d], int(d == a), int(d == b)) for d in range(3)]
            S[a][b] = k3(*fac)
    N = S[0][0].shape[0]
    A = np.zeros((3 * N, 3 * N))
    tr = S[0][0] + S[1][1] + S[2][2]
    for c in range(3):
        for d in range(3):
            blk = lam * S[c][d] + mu * S[d][c]
            if c == d:
                blk = blk + mu * tr
            A[c * N:(c + 1) * N, d * N:(d + 1) * N] = blk
    return A


# ---------------------------------------------------------------------------------------
# Element-level pins
# ---------------------------------------------------------------------------------------

@pytest.mark.parametrize("q", [2, 3])
def test_q1_element_exact(q):
    lam, mu = 1.3, 0.7
    Kex = np.array(q1_element_matrix_sympy(sp.Rational(13, 10), sp.Rational(7, 10)).evalf(20), dtype=float)
    V = synth.uniform_vertices(1, 1, 1, 1.0, 1.0, 1.0)
    tables = E.reference_tables(1, q)
    K = E.element_stiffness(V[0:2, 0:2, 0:2], lam, mu, tables)
    assert np.allclose(K, Kex, atol=1e-15, rtol=0)
    # SURVEY Appendix B.1 closed forms (lexicographic nodes, component-blocked)
    n = 8
    assert abs(K[0, 0] - (lam + 4 * mu) / 9) < 1e-15
    assert abs(K[0, 1] - (-(lam + mu) / 9)) < 1e-15
    assert abs(K[0, n + 1] - (lam - mu) / 12) < 1e-15
    assert abs(K[0, 7] - (-lam / 36 - mu / 9)) < 1e-15
    assert abs(K[0, n + 3] - (-(lam + mu) / 12)) < 1e-15
    assert abs(np.trace(K) - (8 * lam / 3 + 32 * mu / 3)) < 1e-14
    assert abs((K ** 2).sum() - 10 * (7 * lam ** 2 + 11 * lam * mu + 22 * mu ** 2) / 27) < 1e-13


def test_q1_element_eigenvalues():
    V = synth.uniform_vertices(1, 1, 1, 1.0, 1.0, 1.0)
    K = E.element_stiffness(V[0:2, 0:2, 0:2], 1.0, 1.0, E.reference_tables(1, 2))
    ev = np.sort(np.linalg.eigvalsh(K))
    expect = sorted([0] * 6 + [5 / 18] * 3 + [1 / 6] * 2 + [1 / 2] * 3 + [2 / 3] + [5 / 6] * 3 + [1] * 5 + [5 / 2])
    assert np.allclose(ev, expect, atol=1e-14)


def test_element_scaling_with_h():
    """Affine cube of size h: K(h) = h K(1)."""
    tables = E.reference_tables(2, 4)
    V1 = synth.uniform_vertices(1, 1, 1, 1.0, 1.0, 1.0)[0:2, 0:2, 0:2]
    K1 = E.element_stiffness(V1, 1.2, 0.8, tables)
    Kh = E.element_stiffness(0.25 * V1 + 3.0, 1.2, 0.8, tables)
    assert np.allclose(Kh, 0.25 * K1, atol=1e-14)


# ---------------------------------------------------------------------------------------
# Global operator pins
# ---------------------------------------------------------------------------------------

@pytest.mark.parametrize("p,dims,lengths", [
    (1, (2, 3, 2), (1.0, 1.5, 0.7)),
    (2, (2, 2, 2), (1.0, 1.0, 1.0)),
    (3, (2, 1, 2), (0.6, 1.0, 1.3)),
    (4, (1, 2, 1), (1.0, 0.8, 1.0)),
])
@pytest.mark.parametrize("dq", [1, 2])
def test_affine_operator_equals_kronecker(p, dims, lengths, dq):
    nx, ny, nz = dims
    lam, mu = 1.7, 0.45
    P = synth.make_problem("t", nx, ny, nz, p, p + dq, lengths=lengths, lam=lam, mu=mu, seed=5)
    A = oracle.assemble_dense(mesh_of(P))
    Ak = kron_operator(nx, ny, nz, *lengths, p, lam, mu)
    assert np.abs(A - Ak).max() <= 1e-12 * np.abs(Ak).max()   # monomial-basis integration rounding


def _frac_1d(ne, h):
    """Exact 1D matrices for p=2 GLL nodes {0, 1/2, 1} in Fractions."""
    # cardinal polynomials as coefficient lists (ascending) with Fraction coefficients
    def poly_mul(a, b):
        out = [Fraction(0)] * (len(a) + len(b) - 1)
        for i, x in enumerate(a):
            for j, y in enumerate(b):
                out[i + j] += x * y
        return out
    nodes = [Fraction(0), Fraction(1, 2), Fraction(1)]
    L = []
    for i, xi in enumerate(nodes):
        c = [Fraction(1)]
        for j, xj in enumerate(nodes):
            if j != i:
                c = poly_mul(c, [-xj / (xi - xj), 1 / (xi - xj)])
        L.append(c)
    dL = [[k * c[k] for k in range(1, len(c))] for c in L]
    integ = lambda c: sum(ck / (k + 1) for k, ck in enumerate(c))
    m = [[integ(poly_mul(L[a], L[b])) for b in range(3)] for a in range(3)]
    k = [[integ(poly_mul(dL[a], dL[b])) for b in range(3)] for a in range(3)]
    cc = [[integ(poly_mul(dL[a], L[b])) for b in range(3)] for a in range(3)]
    N = 2 * ne + 1
    Z = lambda: np.full((N, N), Fraction(0), dtype=object)
    M, K, C = Z(), Z(), Z()
    for e in range(ne):
        for a in range(3):
            for b in range(3):
                M[2 * e + a, 2 * e + b] += h * m[a][b]
                K[2 * e + a, 2 * e + b] += k[a][b] / h
                C[2 * e + a, 2 * e + b] += cc[a][b]
    return M, K, C


def test_config1_exact_rational_pins():
    """Config 1 (2^3 unit cube, Q2, q=4, lam=mu=1): A is exactly rational.

    Re-derive trace and Frobenius norm in exact Fractions by the Kronecker construction, check
    them against the golden values, then check the oracle (floating point) against them.
    """
    with open(os.path.join(GOLDEN, "config1_exact.json")) as f:
        gold = json.load(f)
    M, K, C = _frac_1d(2, Fraction(1, 2))
    k3 = lambda a, b, c: np.kron(c, np.kron(b, a))
    f1 = lambda d, dI, dJ: {(0, 0): M, (1, 1): K, (1, 0): C, (0, 1): C.T}[(dI, dJ)]
    S = [[k3(*[f1(d, int(d == a), int(d == b)) for d in range(3)]) for b in range(3)] for a in range(3)]
    tr = S[0][0] + S[1][1] + S[2][2]
    trace = Fraction(0)
    fro = Fraction(0)
    diag = []
    for c in range(3):
        for d in range(3):
            blk = S[c][d] + S[d][c] + (tr if c == d else 0)
            fro += sum(v * v for v in blk.ravel())
            if c == d:
                dg = list(np.diag(blk))
                trace += sum(dg)
                diag += dg
    assert trace == Fraction(gold["trace"])
    assert fro == Fraction(gold["frobenius_sq"])
    assert min(diag) == Fraction(gold["diag_min"]) and max(diag) == Fraction(gold["diag_max"])
    # the oracle in floating point
    P = synth.make_config(1)
    A = oracle.assemble_dense(mesh_of(P))
    assert A.shape == (gold["n_dof"], gold["n_dof"])
    assert abs(np.trace(A) - float(trace)) < 1e-12
    assert abs((A ** 2).sum() - float(fro)) < 1e-11
    assert np.count_nonzero(np.abs(A) > 1e-14) == gold["structural_nonzeros"]
    ev = np.linalg.eigvalsh(A)
    assert np.sum(np.abs(ev) < 1e-12) == 6
    assert abs(ev.max() - gold["lambda_max"]) < 1e-12
    assert abs(np.sort(ev)[6] - gold["lambda_min_nonzero"]) < 1e-12
    X = oracle.node_coordinates(mesh_of(P))
    N = X.shape[0]
    u = np.concatenate([X[:, 0], np.zeros(N), np.zeros(N)])
    assert abs(u @ A @ u - gold["energy_u_x"]) < 1e-12
    r = np.concatenate([X[:, 1], -X[:, 0], np.zeros(N)])
    assert np.abs(A @ r).max() < 1e-13


def rigid_modes(X):
    N = X.shape[0]
    z, o = np.zeros(N), np.ones(N)
    x, y, w = X[:, 0], X[:, 1], X[:, 2]
    return [np.concatenate(v) for v in (
        (o, z, z), (z, o, z), (z, z, o),
        (-y, x, z), (z, -w, y), (w, z, -x))]


@pytest.mark.parametrize("p,dq", [(1, 1), (1, 2), (2, 2), (3, 1), (3, 2), (4, 2)])
def test_rigid_modes_perturbed(p, dq):
    P = synth.make_problem("t", 2, 2, 1, p, p + dq, perturb=True, lognormal_material=True, seed=11)
    m = mesh_of(P)
    X = oracle.node_coordinates(m)
    diag_max = None
    for r in rigid_modes(X):
        y = oracle.apply(m, r)
        if diag_max is None:
            A = oracle.assemble_dense(m)
            diag_max = np.abs(np.diag(A)).max()
        assert np.linalg.norm(y) <= 1e-12 * diag_max * np.linalg.norm(r)


@pytest.mark.parametrize("p,dims", [(2, (2, 2, 2)), (3, (2, 1, 2))])
def test_symmetry_psd_nullity(p, dims):
    P = synth.make_problem("t", *dims, p, p + 2, perturb=True, lognormal_material=True, seed=3)
    A = oracle.assemble_dense(mesh_of(P))
    assert np.abs(A - A.T).max() <= 1e-14 * np.abs(A).max()
    ev = np.linalg.eigvalsh(A)
    scale = ev.max()
    assert ev.min() > -1e-13 * scale
    assert np.sum(ev < 1e-11 * scale) == 6


@pytest.mark.parametrize("p", [1, 2, 3])
def test_patch_test_energy(p):
    """u = E X + c at the nodes: u^T A u = Vol (lam tr(eps)^2 + 2 mu eps:eps), constant material."""
    lam, mu = 1.4, 0.6
    P = synth.make_problem("t", 2, 2, 2, p, p + 2, lengths=(1.0, 1.2, 0.9), perturb=True,
                           lam=lam, mu=mu, seed=8)
    m = mesh_of(P)
    X = oracle.node_coordinates(m)
    rng = np.random.default_rng(0)
    G = rng.standard_normal((3, 3))
    c = rng.standard_normal(3)
    U = X @ G.T + c                          # u_i = G_ij X_j + c_i
    u = np.concatenate([U[:, 0], U[:, 1], U[:, 2]])
    eps = 0.5 * (G + G.T)
    vol = 1.0 * 1.2 * 0.9
    expect = vol * (lam * np.trace(eps) ** 2 + 2 * mu * np.sum(eps * eps))
    got = u @ oracle.apply(m, u)
    assert abs(got - expect) <= 1e-13 * abs(expect)


@pytest.mark.parametrize("p,q", [(2, 3), (3, 5), (4, 6)])
def test_interior_equilibrium(p, q):
    """Affine u, constant material: (A u)_i = 0 at every interior dof (exact for q >= (p+2)/2)."""
    P = synth.make_problem("t", 2, 2, 2, p, q, perturb=True, lam=0.9, mu=1.1, seed=21)
    m = mesh_of(P)
    X = oracle.node_coordinates(m)
    G = np.arange(9.0).reshape(3, 3) / 7.0 - 0.3
    U = X @ G.T
    u = np.concatenate([U[:, 0], U[:, 1], U[:, 2]])
    y = oracle.apply(m, u)
    Nx, Ny, Nz = m.node_dims
    K, J, I = np.meshgrid(np.arange(Nz), np.arange(Ny), np.arange(Nx), indexing="ij")
    interior = ((I > 0) & (I < Nx - 1) & (J > 0) & (J < Ny - 1) & (K > 0) & (K < Nz - 1)).reshape(-1)
    interior = np.tile(interior, 3)
    A = oracle.assemble_dense(m)
    assert np.abs(y[interior]).max() <= 1e-13 * np.abs(np.diag(A)).max() * np.abs(u).max()
    assert np.abs(y[~interior]).max() > 1e-3   # boundary tractions are not zero


def test_geometry_affine_and_volume():
    P = synth.make_problem("t", 2, 2, 2, 1, 2, lengths=(1.0, 2.0, 0.5))
    m = mesh_of(P)
    tables = E.reference_tables(1, 2)
    J, detJ, W = E.element_geometry(E.element_vertices(m, 1, 0, 1), tables[2], tables[1])
    assert np.allclose(J, np.diag([0.5, 1.0, 0.25])[None], atol=4e-16, rtol=0)
    assert np.allclose(detJ, 0.125)
    Q = synth.make_problem("t", 3, 2, 2, 2, 4, lengths=(1.0, 2.0, 0.5), perturb=True, seed=2)
    mq = mesh_of(Q)
    tq = E.reference_tables(2, 2)     # det J has degree <= 2 per direction: q=2 is exact
    vol = sum(E.element_geometry(E.element_vertices(mq, ex, ey, ez), tq[2], tq[1])[2].sum()
              for ez in range(2) for ey in range(2) for ex in range(3))
    assert abs(vol - 1.0) < 1e-14


def test_dirichlet_wrapper():
    P = synth.make_problem("t", 2, 2, 2, 2, 4, perturb=True, lognormal_material=True, faces=1 | 32, seed=4)
    m = mesh_of(P)
    Z = oracle.constrained_mask(m)
    Nx, Ny, Nz = m.node_dims
    assert Z.sum() == 3 * (Ny * Nz + Nx * Ny - Ny)           # x=0 face plus z=max face, shared edge once
    idx = np.flatnonzero(Z)[5]
    e = np.zeros(m.num_dofs)
    e[idx] = 1.0
    assert np.array_equal(oracle.apply(m, e), e)               # identity row and column
    rng = np.random.default_rng(1)
    x = rng.uniform(-1, 1, m.num_dofs)
    x[Z] = 0.0
    y = oracle.apply(m, x)
    assert np.all(y[Z] == 0.0)
    # dense: Z A0 Z + (I - Z) with A0 the unconstrained operator
    m0 = oracle.Mesh(m.vertices, m.p, m.q, m.lam, m.mu, 0)
    A0 = oracle.assemble_dense(m0)
    D = np.diag((~Z).astype(float))
    assert np.allclose(oracle.assemble_dense(m), D @ A0 @ D + np.diag(Z.astype(float)), atol=1e-15)


def test_apply_matches_dense_and_rows():
    P = synth.make_problem("t", 3, 2, 2, 3, 5, perturb=True, lognormal_material=True, faces=1, seed=9)
    m = mesh_of(P)
    A = oracle.assemble_dense(m)
    y = oracle.apply(m, P.x)
    assert np.allclose(y, A @ P.x, atol=1e-13 * np.abs(y).max())
    rows = np.random.default_rng(0).choice(m.num_dofs, 200, replace=False)
    rows = np.concatenate([rows, np.flatnonzero(oracle.constrained_mask(m))[:5]])
    yr = oracle.apply_rows(m, P.x, rows)
    assert np.allclose(yr, y[rows], atol=1e-13 * np.abs(y).max(), rtol=0)


def test_config_shapes():
    """DOF / element counts of the BASELINE.json configs."""
    expect = {1: (375, 8), 2: (823_875, 4096), 3: (9_145_875, 13_824), 5: (683_465_475, 1_048_576)}
    for cfg, (ndof, ne) in expect.items():
        P = synth.make_config(cfg, draw_x=False)
        assert (P.num_dofs, P.num_elements) == (ndof, ne)
    ms = [synth.config4_elements(p) for p in range(1, 9)]
    assert ms == [255, 128, 85, 64, 51, 43, 36, 32]
