"""Pins of the paper's analytical models (paper_1709_07122_b200/model.py) to the
numbers PAPER.md itself prints, and to the algebra its §4 comparison states."""
import pytest

from paper_1709_07122_b200 import model

# kron (Fig. 7 caption): n = 33.5 M, m = 1070 M, k = 512, d_i = d_v = 4 B;
# r = 3.06 (Table 6; reading R12).
KRON = dict(n=33.5e6, m=1070e6, k=512)


def test_eq5_kron_is_8_7_gb():
    """Eq. 5 at kron with r = 3.06 predicts ~8.7 GB per iteration (the
    paper measures 10.4 GB)."""
    b = model.pcpm_comm(KRON["n"], KRON["m"], KRON["k"], 3.06)
    assert b == pytest.approx(8.7e9, rel=0.01)


def test_random_access_counts_of_section_4_1():
    """kron with d_v = 4 B, l = 64 B, k = 512: BVGAS_ra ~ 66.9 M, PCPM_ra ~ 0.26 M."""
    assert model.random_accesses("bvgas", m=KRON["m"], d_v=4, l=64) == pytest.approx(66.9e6, rel=1e-3)
    assert model.random_accesses("pcpm", k=KRON["k"]) == pytest.approx(0.26e6, rel=0.01)
    assert model.random_accesses("pdpr", m=1000, c_mr=0.25) == 250
    with pytest.raises(ValueError):
        model.random_accesses("ligra")


def test_eq5_at_r1_matches_bvgas_and_bounds():
    """in the worst case r = 1, PCPM is as good as BVGAS (same m-coefficient
    2(d_i + d_v)), and PCPM_comm lies in [m d_i, m(2 d_i + 2 d_v)] up to the k^2 and n terms."""
    n, m, k = 1e6, 1e8, 8
    small = k * k * 4 + 2 * n * 4
    pc1 = model.pcpm_comm(n, m, k, 1.0)
    assert pc1 - small == pytest.approx(m * (2 * 4 + 2 * 4))
    assert model.bvgas_comm(n, m) - n * (4 + 8) == pytest.approx(m * (2 * 4 + 2 * 4))
    best = model.pcpm_comm(n, m, k, m / n)                      # optimal labelling r = m / n
    assert m * 4 <= best - small <= m * (2 * 4 + 2 * 4)
    # decreasing in r (Fig. 7)
    assert model.pcpm_comm(n, m, k, 5.0) < model.pcpm_comm(n, m, k, 2.0) < pc1


def test_eq3_range_and_breakevens():
    """PDPR_comm in [m d_i, m (d_i + l)] over c_mr in [n d_v / (m l), 1]; Eq. 6 / 7:
    at the break-even c_mr, the m-coefficients of PDPR and BVGAS (resp. PCPM) are equal."""
    n, m, l = 1e6, 1e9, 64
    assert model.pdpr_comm(n, m, 1.0, l=l) == pytest.approx(m * (4 + l) + n * 8)
    lo = model.pdpr_comm(n, m, n * 4 / (m * l), l=l)
    assert lo == pytest.approx(m * 4 + n * 4 + n * 8)
    c6 = model.breakeven_cmr_bvgas(l=l)
    assert c6 == pytest.approx((4 + 8) / 64)
    assert 4 + c6 * l == pytest.approx(2 * (4 + 4))                      # PDPR vs BVGAS per edge
    for r in (1.0, 1.42, 3.06, 7.0):
        c7 = model.breakeven_cmr_pcpm(r, l=l)
        assert c7 == pytest.approx(c6 / r)
        assert 4 + c7 * l == pytest.approx(4 * (1 + 1 / r) + 2 * 4 / r)  # PDPR vs PCPM per edge
