"""The roofline model bench.py reports against the per-element flop
counts SURVEY Appendix A tabulates, and the JSON contract's fixed fields (CPU only)."""

import os
import sys

import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

# flops per element (q = p + 2): total, sum-factorisation part, pointwise part
APPENDIX_A = {1: (7056, 3816, 3240), 2: (22368, 14688, 7680), 3: (55080, 40080, 15000),
              4: (115200, 89280, 25920), 5: (215040, 173880, 41160), 6: (369216, 307776, 61440),
              7: (594648, 507168, 87480), 8: (910560, 790560, 120000)}


@pytest.mark.parametrize("p", range(1, 9))
def test_alg_flops_per_element_match_survey(p):
    tot, sf, pw = APPENDIX_A[p]
    assert bench.alg_flops(p, p + 2, 1) == tot
    assert 120 * (p + 2) ** 3 == pw and tot - pw == sf


def test_config5_counts_and_peak():
    # config 5: 64 x 64 x 256 Q6 hexes, q = 8 (reading R14)
    ne = 64 * 64 * 256
    ndof = 3 * (64 * 6 + 1) ** 2 * (256 * 6 + 1)
    assert ndof == 683465475
    assert bench.alg_flops(6, 8, ne) == 387151036416
    assert bench.alg_bytes(ndof, ne, 8, True) == 16 * ndof + 72 * 512 * ne + 8 * ne
    assert abs(bench.PEAK_FP64_DERIVED - 148 * 64 * 2 * 1.965e9) < 1e6
