"""The paper's analytical traffic models (§4), for reporting.

These are closed-form byte / access counts, not part of the hot path.  bench.py
prints them next to the measured bytes (BASELINE.json north_star: "Bytes actually
moved per iteration are reported next to the paper's communication model, for
both the compressed and the uncompressed bin layout"): Eq. 5 for the PCPM
layouts, Eq. 4 for BVGAS, Eq. 3 for the pull kernel with c_mr measured from its
L2 misses, and the §4.1 random-access counts.  Pinned to the paper's own numbers
(kron: Eq. 5 ~ 8.7 GB, §4.1's 66.9 M / 0.26 M) in tests/test_model.py.
"""
from __future__ import annotations


def pdpr_comm(n: float, m: float, c_mr: float, l: float = 64, d_i: float = 4, d_v: float = 4) -> float:
    """Eq. 3: m(d_i + c_mr l) + n(d_i + d_v)."""
    return m * (d_i + c_mr * l) + n * (d_i + d_v)


def bvgas_comm(n: float, m: float, d_i: float = 4, d_v: float = 4) -> float:
    """Eq. 4: 2m(d_i + d_v) + n(d_i + 2 d_v)."""
    return 2 * m * (d_i + d_v) + n * (d_i + 2 * d_v)


def pcpm_comm(n: float, m: float, k: float, r: float, d_i: float = 4, d_v: float = 4) -> float:
    """Eq. 5: m(d_i(1 + 1/r) + 2 d_v / r) + k^2 d_i + 2 n d_v."""
    return m * (d_i * (1 + 1 / r) + 2 * d_v / r) + k * k * d_i + 2 * n * d_v


def breakeven_cmr_bvgas(l: float = 64, d_i: float = 4, d_v: float = 4) -> float:
    """Eq. 6: BVGAS beats PDPR when c_mr > (d_i + 2 d_v) / l."""
    return (d_i + 2 * d_v) / l


def breakeven_cmr_pcpm(r: float, l: float = 64, d_i: float = 4, d_v: float = 4) -> float:
    """Eq. 7: PCPM beats PDPR when c_mr > (d_i + 2 d_v) / (r l)."""
    return (d_i + 2 * d_v) / (r * l)


def random_accesses(engine: str, m: float = 0, k: float = 0, c_mr: float = 1, l: float = 64,
                    d_v: float = 4) -> float:
    """Leading terms of §4.1: PDPR m c_mr, BVGAS m d_v / l, PCPM k^2."""
    if engine == "pdpr":
        return m * c_mr
    if engine == "bvgas":
        return m * d_v / l
    if engine == "pcpm":
        return k * k
    raise ValueError(engine)
