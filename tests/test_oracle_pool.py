"""The parallel row helper returns oracle.apply_rows (it only splits the rows; the element rows
are then evaluated in different batch shapes, so equality is to rounding)."""

import numpy as np

import oracle
import synth
from tests import oracle_pool


def test_pool_equals_serial_apply_rows():
    P = synth.make_problem("t", 3, 2, 2, 2, 4, perturb=True, lognormal_material=True, faces=1 | 32, seed=4)
    lam, mu = P.material_arrays()
    m = oracle.Mesh(P.vertex_array(), P.p, P.q, lam, mu, P.dirichlet_faces)
    rows = np.random.default_rng(0).choice(P.num_dofs, 400, replace=False)
    serial = oracle.apply_rows(m, P.x, rows)
    par = oracle_pool.apply_rows(m, P.x, rows, procs=3)
    assert np.abs(par - serial).max() <= 1e-14 * np.abs(serial).max()
    assert np.allclose(serial, oracle.apply(m, P.x)[rows], rtol=0, atol=1e-13 * np.abs(serial).max())
