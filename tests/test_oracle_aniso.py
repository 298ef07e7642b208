"""Pins for the oracle's general anisotropic operator (Eq. 2; Voigt
convention of PAPER.md:162), no GPU:

* isotropic Voigt matrix (Eq. 3)  ->  exactly the isotropic operator
* affine box, constant C: equals the independent Kronecker assembly A_cd = sum_kl C_ckdl S_kl
  of exactly integrated 1D matrices (no quadrature, no geometry code)
* rigid-body null space, symmetry, PSD and nullity 6 on perturbed meshes with per-element C
* patch test: u^T A u = sum_e Vol_e eps_v^T C_e eps_v for affine u (engineering shear)
"""

import numpy as np
import pytest

import oracle
import synth
from oracle.elasticity import VOIGT
from tests.test_oracle_operator import mesh_of, one_d_global, rigid_modes


def aniso_mesh(P, C6):
    lam, mu = P.material_arrays()
    return oracle.Mesh(P.vertex_array(), P.p, P.q, lam, mu, P.dirichlet_faces, C6=C6)


@pytest.mark.parametrize("p", [1, 2, 3])
def test_isotropic_voigt_matrix_reduces_to_hooke(p):
    P = synth.make_problem("t", 2, 2, 2, p, p + 2, perturb=True, lognormal_material=True, seed=p)
    lam, mu = P.material_arrays()
    C6 = np.stack([[[synth.isotropic_C6(lam[k, j, i], mu[k, j, i]) for i in range(2)] for j in range(2)]
                   for k in range(2)])
    A_iso = oracle.assemble_dense(mesh_of(P))
    A_ani = oracle.assemble_dense(aniso_mesh(P, C6))
    assert np.abs(A_ani - A_iso).max() <= 1e-13 * np.abs(A_iso).max()


@pytest.mark.parametrize("p,dims,lengths", [(1, (2, 3, 2), (1.0, 1.5, 0.7)), (2, (2, 1, 2), (0.6, 1.0, 1.3)),
                                            (3, (1, 2, 1), (1.0, 0.8, 1.0))])
def test_affine_box_equals_kronecker(p, dims, lengths):
    rng = np.random.default_rng(11 + p)
    C6 = synth.random_C6(rng, ())
    P = synth.make_problem("t", *dims, p, p + 1, lengths=lengths, seed=2)
    A = oracle.assemble_dense(aniso_mesh(P, C6))
    nodes = oracle.gll_nodes(p)
    mats = [one_d_global(nodes, n, L / n) for n, L in zip(dims, lengths)]
    k3 = lambda a, b, c: np.kron(c, np.kron(b, a))
    f1 = lambda M, K, C, dI, dJ: {(0, 0): M, (1, 1): K, (1, 0): C, (0, 1): C.T}[(dI, dJ)]
    S = [[k3(*[f1(*mats[d], int(d == a), int(d == b)) for d in range(3)]) for b in range(3)] for a in range(3)]
    N = S[0][0].shape[0]
    Ak = np.zeros((3 * N, 3 * N))
    for c in range(3):
        for d in range(3):
            blk = sum(C6[VOIGT[c, k], VOIGT[d, l]] * S[k][l] for k in range(3) for l in range(3))
            Ak[c * N:(c + 1) * N, d * N:(d + 1) * N] = blk
    assert np.abs(A - Ak).max() <= 1e-12 * np.abs(Ak).max()


@pytest.mark.parametrize("p", [1, 2, 3])
def test_rigid_modes_symmetry_nullity(p):
    P = synth.make_problem("t", 2, 2, 2, p, p + 2, perturb=True, seed=20 + p)
    C6 = synth.random_C6(np.random.default_rng(p), (2, 2, 2))
    m = aniso_mesh(P, C6)
    A = oracle.assemble_dense(m)
    X = oracle.node_coordinates(m)
    R = np.stack(rigid_modes(X), axis=1)
    scale = np.abs(A).max()
    assert np.abs(A @ R).max() <= 1e-11 * scale * np.abs(R).max()
    assert np.abs(A - A.T).max() <= 1e-13 * scale
    ev = np.linalg.eigvalsh(A)
    assert ev.min() >= -1e-10 * scale
    assert np.sum(ev < 1e-9 * ev.max()) == 6


@pytest.mark.parametrize("p", [1, 2])
def test_patch_energy(p):
    P = synth.make_problem("t", 2, 2, 2, p, p + 2, perturb=True, seed=30 + p)
    rng = np.random.default_rng(5)
    C6 = synth.random_C6(rng, (2, 2, 2))
    m = aniso_mesh(P, C6)
    A = oracle.assemble_dense(m)
    X = oracle.node_coordinates(m)
    E = rng.normal(size=(3, 3))
    u = np.concatenate([X @ E[c] for c in range(3)])
    eps = 0.5 * (E + E.T)
    ev = np.array([eps[0, 0], eps[1, 1], eps[2, 2], 2 * eps[1, 2], 2 * eps[0, 2], 2 * eps[0, 1]])
    # element volumes from the exact trilinear map (q >= 2 integrates det J exactly)
    Gref, w3, g = oracle.elasticity.reference_tables(p, p + 2)
    vols = np.zeros((2, 2, 2))
    for k in range(2):
        for j in range(2):
            for i in range(2):
                _, _, W = oracle.elasticity.element_geometry(oracle.elasticity.element_vertices(m, i, j, k), g, w3)
                vols[k, j, i] = W.sum()
    expect = sum(vols[k, j, i] * ev @ C6[k, j, i] @ ev for k in range(2) for j in range(2) for i in range(2))
    assert abs(u @ A @ u - expect) <= 1e-12 * abs(expect)


@pytest.mark.parametrize("p", [1, 2])
def test_aniso_diagonal_equals_assembled(p):
    P = synth.make_problem("t", 2, 2, 2, p, p + 2, perturb=True, faces=1, seed=40 + p)
    m = aniso_mesh(P, synth.random_C6(np.random.default_rng(7), (2, 2, 2)))
    d = oracle.diagonal(m)
    A = oracle.assemble_dense(m)
    assert np.abs(d - np.diag(A)).max() <= 1e-13 * np.abs(d).max()
