"""CPU-side checks of the C-ABI library (no compute calls, no GPU needed)."""

import ctypes
import re
import os

import numpy as np
import pytest

from oracle import rules
from tests.conftest import cuda_available

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "elas.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(elas_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol(lib):
    names = header_functions()
    assert "elas_create" in names and "elas_apply" in names and "elas_destroy" in names
    for n in names:
        assert hasattr(lib, n), f"libelas.so does not export {n}"
        assert ctypes.cast(getattr(lib, n), ctypes.c_void_p).value


def test_binding_names_match_header():
    from paper_2601_08374_b200 import elas
    assert sorted(elas.EXPORTED) == header_functions()
    for n in header_functions():
        assert callable(getattr(elas, n))


def test_slab_range():
    from paper_2601_08374_b200 import elas
    for nz, P in [(256, 1), (256, 2), (256, 8), (255, 8), (7, 3), (3, 3)]:
        covered = []
        for r in range(P):
            b, e = elas.elas_slab_range(nz, r, P)
            assert b == (r * nz) // P and e == ((r + 1) * nz) // P and e > b
            covered += list(range(b, e))
        assert covered == list(range(nz))
    for bad in [(4, 0, 8), (8, 8, 8), (8, -1, 2), (8, 0, 0)]:
        with pytest.raises(Exception):
            elas.elas_slab_range(*bad)


@pytest.mark.parametrize("p", range(1, 9))
def test_host_tables_match_oracle_tables(p):
    """The library's barycentric tables vs the oracle's product-formula tables (independent code)."""
    from paper_2601_08374_b200 import elas
    for q in (p + 1, p + 2, 1, 3):
        nodes, g, w, B, D = elas.elas_tables(p, q)
        go, wo = rules.gauss_legendre(q)
        no = rules.gll_nodes(p)
        assert np.allclose(nodes, no, atol=2e-16, rtol=0)
        assert np.allclose(g, go, atol=2e-16, rtol=0)
        assert np.allclose(w, wo, atol=5e-16, rtol=0)
        assert np.allclose(B, rules.lagrange_values(no, go), atol=5e-15, rtol=0)
        assert np.allclose(D, rules.lagrange_derivatives(no, go), atol=1e-13 * max(1, p * p), rtol=0)


def test_tables_coincident_point():
    """q=3 Gauss point 1/2 coincides with the p=2 GLL midpoint: differentiation-matrix branch."""
    from paper_2601_08374_b200 import elas
    nodes, g, w, B, D = elas.elas_tables(2, 3)
    assert g[1] == 0.5 and nodes[1] == 0.5
    assert np.array_equal(B[1], [0.0, 1.0, 0.0])
    assert np.allclose(D[1], [-1.0, 0.0, 1.0], atol=1e-15)


def test_invalid_arguments_fail_loudly():
    from paper_2601_08374_b200 import elas
    with pytest.raises(elas.ElasError, match="p must be"):
        elas.elas_create(2, 2, 2, 9, 10, 1.0, 1.0)
    with pytest.raises(elas.ElasError, match="q must be"):
        elas.elas_create(2, 2, 2, 2, 7, 1.0, 1.0)
    with pytest.raises(elas.ElasError, match=">= 1"):
        elas.elas_create(0, 2, 2, 2, 4, 1.0, 1.0)
    with pytest.raises(elas.ElasError):
        elas.elas_tables(0, 3)


@pytest.mark.skipif(cuda_available(), reason="checks the no-GPU behaviour")
def test_create_without_gpu_fails_loudly():
    """No CPU fallback: without a device the library reports a CUDA error instead of computing."""
    from paper_2601_08374_b200 import elas
    with pytest.raises(elas.ElasError, match="cuda|CUDA"):
        elas.elas_create(2, 2, 2, 2, 4, 1.0, 1.0)


def test_invalid_material_rejected_before_any_device_work():
    from paper_2601_08374_b200 import elas
    with pytest.raises(elas.ElasError, match="material"):
        elas.elas_create(2, 2, 2, 2, 4, 1.0, 0.0)
    with pytest.raises(elas.ElasError, match="material"):
        elas.elas_create(2, 2, 2, 2, 4, -1.0, 1.0)       # 3 lam + 2 mu < 0
    lam = np.ones((2, 2, 2))
    mu = np.ones((2, 2, 2))
    mu[1, 0, 1] = -0.5
    with pytest.raises(elas.ElasError, match="element 5"):
        elas.elas_create(2, 2, 2, 2, 4, lam, mu)


def test_gmg_slab_alignment_rejected_before_any_device_work():
    """Z-slab GMG needs every level's slabs aligned: nz divisible by nranks * 2^(levels-1)."""
    from paper_2601_08374_b200 import elas
    with pytest.raises(elas.ElasError, match="nranks"):
        elas.elas_gmg_create(2, 2, 12, 2, 4, 1.0, 1.0, levels=3, rank=0, nranks=2)   # 12 % 8 != 0
    with pytest.raises(elas.ElasError, match="divisible"):
        elas.elas_gmg_create(2, 3, 8, 2, 4, 1.0, 1.0, levels=2)                       # ny odd


def test_gmg_rejects_single_level():
    """elas_gmg_create needs levels >= 2: with one level the coarse PCG would run on the finest
    op and share its work vectors with the outer elas_pcg_gmg.  The argument check
    precedes every CUDA call, so this runs without a GPU."""
    from paper_2601_08374_b200 import elas
    lam = np.ones(8)
    with pytest.raises(elas.ElasError, match="levels >= 2"):
        elas.elas_gmg_create(2, 2, 2, 2, 4, lam, lam, levels=1)
