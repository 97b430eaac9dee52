"""CPU oracle for the PCPM PageRank / SpMV hot path (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
and ``--impl reference`` legs may import this package.  The product package
``paper_1709_07122_b200`` never imports it, and the two share no code.

The arithmetic lives in ``pcpm_oracle.c`` (plain fp64 C, each function citing
the PAPER.md passage it follows); this module only marshals numpy arrays into
it through ctypes.  ``build_oracle()`` compiles the C file with gcc.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "pcpm_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build_oracle(force: bool = False) -> str:
    """Compile oracle/pcpm_oracle.c into oracle/liboracle.so (gcc -O2 -fopenmp)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build_oracle()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        lib.oracle_num_threads.restype = ctypes.c_int
        lib.oracle_transpose.argtypes = [I64, P, P, P, P]
        lib.oracle_pagerank_pull.argtypes = [I64, P, P, P, ctypes.c_double, ctypes.c_int, P]
        lib.oracle_pagerank_pull_step.argtypes = [I64, P, P, P, ctypes.c_double, P, P]
        lib.oracle_pagerank.argtypes = [I64, P, P, ctypes.c_double, ctypes.c_int, P]
        lib.oracle_pagerank_weighted.argtypes = [I64, P, P, P, ctypes.c_double, ctypes.c_int, P]
        lib.oracle_spmv_t.argtypes = [I64, I64, P, P, P, P, P]
        lib.oracle_layout_sizes.argtypes = [I64, I64, P, P, ctypes.c_int, P, P, P]
        lib.oracle_layout.argtypes = [I64, I64, P, P, P, ctypes.c_int, P, P, P, P, P, P, P]
        lib.oracle_scatter.argtypes = [I64, I64, P, P, P, P, P]
        lib.oracle_gather.argtypes = [I64, I64, P, P, P, P, P, P]
        for f in ("oracle_transpose", "oracle_pagerank_pull", "oracle_pagerank_pull_step", "oracle_pagerank", "oracle_pagerank_weighted",
                  "oracle_spmv_t",
                  "oracle_layout_sizes", "oracle_layout", "oracle_scatter", "oracle_gather"):
            getattr(lib, f).restype = ctypes.c_int
        _lib = lib
    return _lib


def _p(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def _csr(row_ptr, col):
    row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
    col = np.ascontiguousarray(col, dtype=np.uint32)
    if col.size == 0:
        col = np.zeros(1, dtype=np.uint32)[:0]
    return row_ptr, col


def num_threads() -> int:
    return int(_load().oracle_num_threads())


def set_threads(t: int) -> None:
    """OpenMP threads of the oracle's parallel loops (timing only; results do not depend on it)."""
    _load().oracle_set_threads(int(t))


def transpose(n, row_ptr, col):
    """In-adjacency (CSC) of the CSR graph: (in_ptr int64[n+1], in_src uint32[m])."""
    row_ptr, col = _csr(row_ptr, col)
    m = int(row_ptr[n])
    in_ptr = np.zeros(n + 1, dtype=np.int64)
    in_src = np.zeros(max(m, 1), dtype=np.uint32)
    rc = _load().oracle_transpose(n, _p(row_ptr), _p(col), _p(in_ptr), _p(in_src))
    if rc:
        raise ValueError(f"oracle_transpose failed ({rc})")
    return in_ptr, in_src[:m]


def pagerank_pull(n, row_ptr, in_ptr, in_src, d=0.85, iters=20):
    """Eq. 1 in pull form (Alg. 1) given a precomputed CSC; returns float64[n]."""
    row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
    in_ptr = np.ascontiguousarray(in_ptr, dtype=np.int64)
    in_src = np.ascontiguousarray(in_src, dtype=np.uint32)
    if in_src.size == 0:
        in_src = np.zeros(1, dtype=np.uint32)
    pr = np.zeros(n, dtype=np.float64)
    rc = _load().oracle_pagerank_pull(n, _p(row_ptr), _p(in_ptr), _p(in_src), float(d), int(iters), _p(pr))
    if rc:
        raise ValueError(f"oracle_pagerank_pull failed ({rc})")
    return pr


class PullState:
    """Caller-owned state for stepping the pull oracle one Eq. 1 update at a time
    (oracle_pagerank_pull_step): PR_t and 3n doubles of scratch, allocated once."""

    def __init__(self, n, row_ptr, in_ptr, in_src):
        self.n = n
        self.row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
        self.in_ptr = np.ascontiguousarray(in_ptr, dtype=np.int64)
        self.in_src = np.ascontiguousarray(in_src, dtype=np.uint32)
        if self.in_src.size == 0:
            self.in_src = np.zeros(1, dtype=np.uint32)
        self.pr = np.full(n, 1.0 / n, dtype=np.float64)             # PR_0 (R2)
        self.work = np.zeros(3 * n, dtype=np.float64)

    def step(self, d=0.85):
        rc = _load().oracle_pagerank_pull_step(self.n, _p(self.row_ptr), _p(self.in_ptr), _p(self.in_src), float(d),
                                                _p(self.pr), _p(self.work))
        if rc:
            raise ValueError(f"oracle_pagerank_pull_step failed ({rc})")
        return self.pr


def pagerank(n, row_ptr, col, d=0.85, iters=20):
    """PageRank by Eq. 1 with uniform dangling redistribution (R1); float64[n]."""
    row_ptr, col = _csr(row_ptr, col)
    pr = np.zeros(n, dtype=np.float64)
    colp = col if col.size else np.zeros(1, dtype=np.uint32)
    rc = _load().oracle_pagerank(n, _p(row_ptr), _p(colp), float(d), int(iters), _p(pr))
    if rc:
        raise ValueError(f"oracle_pagerank failed ({rc})")
    return pr


def pagerank_weighted(n, row_ptr, col, w, d=0.85, iters=20):
    """Weighted PageRank (reading R24): u passes PR(u) w(u,v)/W(u) to v; float64[n]."""
    row_ptr, col = _csr(row_ptr, col)
    w = np.ascontiguousarray(w, dtype=np.float32)
    pr = np.zeros(n, dtype=np.float64)
    colp = col if col.size else np.zeros(1, dtype=np.uint32)
    wp = w if w.size else np.zeros(1, dtype=np.float32)
    rc = _load().oracle_pagerank_weighted(n, _p(row_ptr), _p(colp), _p(wp), float(d), int(iters), _p(pr))
    if rc:
        raise ValueError(f"oracle_pagerank_weighted failed ({rc})")
    return pr


def spmv_t(n_src, n_dst, row_ptr, col, val, x):
    """y[v] = sum_{(u,v) in CSR} val(u,v) * x[u] in fp64 (y = M^T x, Eq. 2 orientation)."""
    row_ptr, col = _csr(row_ptr, col)
    colp = col if col.size else np.zeros(1, dtype=np.uint32)
    val = None if val is None else np.ascontiguousarray(val, dtype=np.float32)
    if val is not None and val.size == 0:
        val = np.zeros(1, dtype=np.float32)
    x = np.ascontiguousarray(x, dtype=np.float32)
    y = np.zeros(max(n_dst, 1), dtype=np.float64)
    rc = _load().oracle_spmv_t(n_src, n_dst, _p(row_ptr), _p(colp), _p(val), _p(x), _p(y))
    if rc:
        raise ValueError(f"oracle_spmv_t failed ({rc})")
    return y[:n_dst]


@dataclass
class Layout:
    n_src: int
    n_dst: int
    b: int
    k_src: int
    k_dst: int
    e_prime: int
    ids: np.ndarray            # uint32[m]
    png_src: np.ndarray        # uint32[E']
    png_off: np.ndarray        # uint64[k_src, k_dst+1]
    upd_off: np.ndarray        # uint64[k_src, k_dst]
    bin_id_start: np.ndarray   # uint64[k_dst+1]
    bin_upd_start: np.ndarray  # uint64[k_dst+1]
    w: np.ndarray | None       # float32[m] (weights aligned with ids) or None


def layout(n_src, n_dst, row_ptr, col, b, val=None, with_weights=False):
    """The PCPM bins + PNG layout by plain definition."""
    row_ptr, col = _csr(row_ptr, col)
    colp = col if col.size else np.zeros(1, dtype=np.uint32)
    lib = _load()
    k_src = ctypes.c_int64()
    k_dst = ctypes.c_int64()
    ep = ctypes.c_int64()
    lib.oracle_layout_sizes(n_src, n_dst, _p(row_ptr), _p(colp), int(b), ctypes.byref(k_src),
                            ctypes.byref(k_dst), ctypes.byref(ep))
    ks, kd, e = k_src.value, k_dst.value, ep.value
    m = int(row_ptr[n_src])
    ids = np.zeros(max(m, 1), dtype=np.uint32)
    png_src = np.zeros(max(e, 1), dtype=np.uint32)
    png_off = np.zeros(max(ks * (kd + 1), 1), dtype=np.uint64)
    upd_off = np.zeros(max(ks * kd, 1), dtype=np.uint64)
    bis = np.zeros(kd + 1, dtype=np.uint64)
    bus = np.zeros(kd + 1, dtype=np.uint64)
    want_w = with_weights or val is not None
    w = np.zeros(max(m, 1), dtype=np.float32) if want_w else None
    valp = None if val is None else np.ascontiguousarray(val, dtype=np.float32)
    if valp is not None and valp.size == 0:
        valp = np.zeros(1, dtype=np.float32)
    rc = lib.oracle_layout(n_src, n_dst, _p(row_ptr), _p(colp), _p(valp), int(b), _p(ids), _p(png_src),
                           _p(png_off), _p(upd_off), _p(bis), _p(bus), _p(w))
    if rc:
        raise ValueError(f"oracle_layout failed ({rc})")
    return Layout(n_src, n_dst, b, ks, kd, e, ids[:m], png_src[:e],
                  png_off[:ks * (kd + 1)].reshape(ks, kd + 1), upd_off[:ks * kd].reshape(ks, kd),
                  bis, bus, None if w is None else w[:m])


def scatter(lay: Layout, x):
    """Alg. 4: upd[upd_off[p][j]+t] = x[png_src[png_off[p][j]+t]] (fp32 copy)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    upd = np.zeros(max(lay.e_prime, 1), dtype=np.float32)
    png_src = lay.png_src if lay.png_src.size else np.zeros(1, dtype=np.uint32)
    png_off = np.ascontiguousarray(lay.png_off, dtype=np.uint64)
    upd_off = np.ascontiguousarray(lay.upd_off, dtype=np.uint64)
    if png_off.size == 0:
        png_off = np.zeros(1, dtype=np.uint64)
    if upd_off.size == 0:
        upd_off = np.zeros(1, dtype=np.uint64)
    xx = x if x.size else np.zeros(1, dtype=np.float32)
    rc = _load().oracle_scatter(lay.k_src, lay.k_dst, _p(png_src), _p(png_off), _p(upd_off), _p(xx), _p(upd))
    if rc:
        raise ValueError(f"oracle_scatter failed ({rc})")
    return upd[:lay.e_prime]


def gather(lay: Layout, upd, w=None):
    """Alg. 5 branch-avoiding gather in fp64: acc[v] = sum of (w *) upd over v's IDs."""
    ids = lay.ids if lay.ids.size else np.zeros(1, dtype=np.uint32)
    upd = np.ascontiguousarray(upd, dtype=np.float32)
    if upd.size == 0:
        upd = np.zeros(1, dtype=np.float32)
    wp = None if w is None else np.ascontiguousarray(w, dtype=np.float32)
    if wp is not None and wp.size == 0:
        wp = np.zeros(1, dtype=np.float32)
    acc = np.zeros(max(lay.n_dst, 1), dtype=np.float64)
    rc = _load().oracle_gather(lay.k_dst, lay.n_dst, _p(ids), _p(upd), _p(wp), _p(lay.bin_id_start),
                               _p(lay.bin_upd_start), _p(acc))
    if rc:
        raise ValueError(f"oracle_gather failed ({rc})")
    return acc[:lay.n_dst]
