"""Pins for the oracle GMG V-cycle (no GPU).  PAPER.md:197-218 (Sec. 3, Fig. 2), SPEC solvers.

* 1D prolongation reproduces every polynomial of degree <= p exactly (finite element
  interpolation, closed form: the polynomial itself) and its rows sum to 1
* 3D prolongation maps an affine coarse field to the same affine fine field
* V-cycle symmetric and positive (SPEC "Preconditioner SPD", symmetric V-cycle)
* 2-level p=1 CG convergence factor <= 0.5 (SPEC gmg_vcycle example)
* GMG-PCG beats Jacobi and Chebyshev-PCG; iterations mesh-independent within 5 (SPEC invariant)
"""

import numpy as np
import pytest

import oracle
import synth
from oracle import gmg
from tests.test_oracle_operator import mesh_of


@pytest.mark.parametrize("p", range(1, 9))
def test_prolongation_1d_polynomial_exactness(p):
    nc = 3
    P = gmg.prolongation_1d(p, nc)
    xi = oracle.gll_nodes(p)
    Xc = np.concatenate([e + xi[:-1] for e in range(nc)] + [[nc]]) / nc
    Xf = np.concatenate([e + xi[:-1] for e in range(2 * nc)] + [[2 * nc]]) / (2 * nc)
    rng = np.random.default_rng(p)
    coef = rng.standard_normal(p + 1)
    f = lambda t: np.polyval(coef, t)
    assert np.abs(P @ f(Xc) - f(Xf)).max() <= 1e-12 * np.abs(f(Xf)).max()
    assert np.abs(P.sum(axis=1) - 1).max() <= 1e-13


@pytest.mark.parametrize("p", [1, 2, 3])
def test_prolongation_3d_affine_field(p):
    P = synth.make_problem("t", 4, 2, 2, p, p + 1, lengths=(1.0, 0.7, 1.3), seed=1)
    fine = mesh_of(P)
    coarse = gmg.coarsen(fine)
    Xf, Xc = oracle.node_coordinates(fine), oracle.node_coordinates(coarse)
    E = np.array([[0.3, -0.2, 0.5], [0.1, 0.4, -0.3], [-0.6, 0.2, 0.25]])
    uc = np.concatenate([Xc @ E[c] + c for c in range(3)])
    uf = np.concatenate([Xf @ E[c] + c for c in range(3)])
    Pm = gmg.prolongation(fine, coarse)
    assert np.abs(Pm @ uc - uf).max() <= 1e-13 * np.abs(uf).max()


def test_coarsen_material_and_geometry():
    P = synth.make_problem("t", 4, 4, 2, 2, 4, perturb=True, lognormal_material=True, seed=3)
    fine = mesh_of(P)
    c = gmg.coarsen(fine)
    assert (c.nx, c.ny, c.nz) == (2, 2, 1)
    assert np.isclose(c.lam[0, 1, 1], fine.lam[0:2, 2:4, 2:4].mean())
    assert np.array_equal(c.vertices[1, 2, 1], fine.vertices[2, 4, 2])
    assert gmg.coarsen(c) is None


def build(p, dims, faces=1, levels=2, seed=5, perturb=True):
    P = synth.make_problem("t", *dims, p, p + 1, perturb=perturb, lognormal_material=perturb, faces=faces, seed=seed)
    return mesh_of(P), gmg.GMG(mesh_of(P), levels)


def test_vcycle_symmetric_positive():
    m, G = build(2, (4, 4, 2), levels=2)
    rng = np.random.default_rng(0)
    x, b = rng.standard_normal((2, m.num_dofs))
    Mx, Mb = G.vcycle(x), G.vcycle(b)
    assert abs(x @ Mb - Mx @ b) <= 1e-10 * np.linalg.norm(x) * np.linalg.norm(Mb)
    for _ in range(5):
        v = rng.standard_normal(m.num_dofs)
        assert v @ G.vcycle(v) > 0
    assert not G.vcycle(np.zeros(m.num_dofs)).any()


def test_two_level_p1_convergence_factor():
    m, G = build(1, (4, 4, 4), levels=2, perturb=False)
    b = synth.splitmix_uniform(m.num_dofs, 1)
    x, it, hist = oracle.pcg(m, b, G.vcycle, 1e-8, 200, matvec=lambda v: G.levels[0].A @ v)
    assert hist[-1] <= 1e-8
    factor = hist[-1] ** (1.0 / it)
    assert factor <= 0.5
    assert np.linalg.norm(G.levels[0].A @ x - b) <= 1e-6 * np.linalg.norm(b)


def test_gmg_beats_one_level_preconditioners():
    m, G = build(2, (4, 4, 4), levels=3)
    A = G.levels[0].A
    mv = lambda v: A @ v
    b = synth.splitmix_uniform(m.num_dofs, 2)
    d = G.levels[0].d
    _, it_g, _ = oracle.pcg(m, b, G.vcycle, 1e-8, 500, matvec=mv)
    _, it_j, _ = oracle.pcg(m, b, lambda r: r / d, 1e-8, 5000, matvec=mv)
    L0 = G.levels[0]
    _, it_c, _ = oracle.pcg(m, b, lambda r: L0.smooth(r, np.zeros_like(r)), 1e-8, 5000, matvec=mv)
    assert it_g < it_c < it_j


@pytest.mark.parametrize("p,dims", [(1, [(4, 4, 4), (8, 8, 8)]), (2, [(2, 2, 2), (4, 4, 4)])])
def test_mesh_independence(p, dims):
    its = []
    for k, dm in enumerate(dims):
        m, G = build(p, dm, levels=2 + k, perturb=False)
        b = synth.splitmix_uniform(m.num_dofs, 3)
        _, it, _ = oracle.pcg(m, b, G.vcycle, 1e-8, 500, matvec=lambda v, A=G.levels[0].A: A @ v)
        its.append(it)
    assert abs(its[1] - its[0]) <= 5
