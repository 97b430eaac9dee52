"""Seeded synthetic graphs shaped like the paper's workloads (BASELINE.json configs).

The paper's datasets (gplus, pld, web, kron, twitter, sd1; Table 4,
P:418-425) are not available here; these generators stand in for them
(DESIGN.md "Inputs"):

  RMAT (R-MAT recursive quadrant choice, the Graph500-style Kronecker shape of
  P:410): for every raw edge e and every level l (most significant bit first)
  a 53-bit uniform r = h(seed, 100 + l, e) >> 11 picks the quadrant
      r < a -> (0,0),  r < a+b -> (0,1),  r < a+b+c -> (1,0),  else (1,1)
  where the pair is (source bit, destination bit).  No noise.  (Reading R17.)
  ER: src = ((h(seed,200,e) >> 32) * n) >> 32, dst likewise with stream 201.
  Random labelling: vertex i gets the rank of h(seed, 300, i) >> 1 (stable).
  Duplicates are removed, self-loops kept (R10).  The CSR lists each row's
  columns strictly increasing.

Everything is a pure function of the seed; the numpy and torch backends give
bit-identical CSR (tests/test_inputs.py).  Large configs use the torch backend
on the GPU (generation is test infrastructure, not the timed path).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .rng import (counter_hash_np, counter_hash_torch, u53_np, u53_torch, top_bits_np,
                  top_bits_torch, _lsr)

S_RMAT = 100
S_ER_SRC, S_ER_DST = 200, 201
S_PERM = 300
S_VAL, S_X = 400, 401

CHUNK = 1 << 25


@dataclass
class GraphCSR:
    """A CSR matrix M (row u lists destinations v; push form).

    ``row_ptr`` int64[n_src+1], ``col`` uint32 (numpy) / int32 bit pattern
    (torch), ``values`` float32 or None.  For PageRank n_src == n_dst.
    """
    name: str
    n_src: int
    n_dst: int
    row_ptr: object
    col: object
    values: object = None
    meta: dict = field(default_factory=dict)

    @property
    def m(self) -> int:
        return int(self.row_ptr[-1])

    @property
    def backend(self) -> str:
        return "np" if isinstance(self.row_ptr, np.ndarray) else "torch"

    def to_numpy(self) -> "GraphCSR":
        if self.backend == "np":
            return self
        rp = self.row_ptr.cpu().numpy().astype(np.int64)
        col = self.col.cpu().numpy().view(np.uint32)
        val = None if self.values is None else self.values.cpu().numpy().astype(np.float32)
        return GraphCSR(self.name, self.n_src, self.n_dst, rp, col, val, dict(self.meta))


def _thresholds(a: float, b: float, c: float):
    s = float(1 << 53)
    return int(a * s), int((a + b) * s), int((a + b + c) * s)


def rmat_edges(scale: int, seed: int, a: float, b: float, c: float, start: int, count: int,
               backend: str = "np", device=None):
    """Raw RMAT edges e in [start, start+count): (src, dst) int64 arrays."""
    ta, tab, tabc = _thresholds(a, b, c)
    if backend == "np":
        e = np.arange(start, start + count, dtype=np.uint64)
        src = np.zeros(count, dtype=np.int64)
        dst = np.zeros(count, dtype=np.int64)
        for lvl in range(scale):
            r = u53_np(counter_hash_np(seed, S_RMAT + lvl, e))
            sb = (r >= tab).astype(np.int64)
            db = (((r >= ta) & (r < tab)) | (r >= tabc)).astype(np.int64)
            bit = scale - 1 - lvl
            src |= sb << bit
            dst |= db << bit
        return src, dst
    import torch
    e = torch.arange(start, start + count, dtype=torch.int64, device=device)
    src = torch.zeros(count, dtype=torch.int64, device=device)
    dst = torch.zeros(count, dtype=torch.int64, device=device)
    for lvl in range(scale):
        r = u53_torch(counter_hash_torch(seed, S_RMAT + lvl, e))
        sb = (r >= tab).to(torch.int64)
        db = (((r >= ta) & (r < tab)) | (r >= tabc)).to(torch.int64)
        bit = scale - 1 - lvl
        src |= sb << bit
        dst |= db << bit
    return src, dst


def er_edges(n: int, seed: int, start: int, count: int, backend: str = "np", device=None):
    """Raw Erdos-Renyi edges: src, dst uniform in [0, n) (n <= 2^31)."""
    if backend == "np":
        e = np.arange(start, start + count, dtype=np.uint64)
        hs = counter_hash_np(seed, S_ER_SRC, e) >> np.uint64(32)
        hd = counter_hash_np(seed, S_ER_DST, e) >> np.uint64(32)
        return ((hs * np.uint64(n)) >> np.uint64(32)).astype(np.int64), \
               ((hd * np.uint64(n)) >> np.uint64(32)).astype(np.int64)
    import torch
    e = torch.arange(start, start + count, dtype=torch.int64, device=device)
    hs = _lsr(counter_hash_torch(seed, S_ER_SRC, e), 32)
    hd = _lsr(counter_hash_torch(seed, S_ER_DST, e), 32)
    return _lsr(hs * n, 32), _lsr(hd * n, 32)


def random_permutation(n: int, seed: int, backend: str = "np", device=None):
    """perm[old] = new label: rank of h(seed, 300, old) >> 1 (stable ties by old id)."""
    if backend == "np":
        keys = (counter_hash_np(seed, S_PERM, np.arange(n, dtype=np.uint64)) >> np.uint64(1)).astype(np.int64)
        order = np.argsort(keys, kind="stable")
        perm = np.empty(n, dtype=np.int64)
        perm[order] = np.arange(n, dtype=np.int64)
        return perm
    import torch
    keys = _lsr(counter_hash_torch(seed, S_PERM, torch.arange(n, dtype=torch.int64, device=device)), 1)
    order = torch.sort(keys, stable=True).indices
    perm = torch.empty(n, dtype=torch.int64, device=device)
    perm[order] = torch.arange(n, dtype=torch.int64, device=device)
    return perm


def unit_values_np(seed: int, stream: int, idx: np.ndarray) -> np.ndarray:
    """float32 values uniform in [-1, 1): 2 * (h >> 40) * 2^-24 - 1 (exact in fp32)."""
    k = top_bits_np(counter_hash_np(seed, stream, idx), 24)
    return (k.astype(np.float64) * (2.0 ** -23) - 1.0).astype(np.float32)


def unit_values_torch(seed: int, stream: int, idx):
    import torch
    k = top_bits_torch(counter_hash_torch(seed, stream, idx), 24)
    return (k.to(torch.float64) * (2.0 ** -23) - 1.0).to(torch.float32)


def edges_to_csr(keys, n_src: int, n_dst: int, backend: str):
    """Sorted unique keys (u << 32 | v) -> (row_ptr int64[n_src+1], col)."""
    if backend == "np":
        keys = np.sort(keys, kind="stable")
        if keys.size:
            keep = np.empty(keys.size, dtype=bool)
            keep[0] = True
            np.not_equal(keys[1:], keys[:-1], out=keep[1:])
            keys = keys[keep]
        rows = keys >> 32
        col = (keys & 0xFFFFFFFF).astype(np.uint32)
        counts = np.bincount(rows, minlength=n_src).astype(np.int64)
        row_ptr = np.zeros(n_src + 1, dtype=np.int64)
        np.cumsum(counts, out=row_ptr[1:])
        return row_ptr, col, keys
    import torch
    keys = torch.unique(keys, sorted=True)
    rows = keys >> 32
    col = (keys & 0xFFFFFFFF).to(torch.int32)   # n < 2^31, so the int32 bit pattern is the u32
    counts = torch.bincount(rows, minlength=n_src)
    row_ptr = torch.zeros(n_src + 1, dtype=torch.int64, device=keys.device)
    torch.cumsum(counts, 0, out=row_ptr[1:])
    return row_ptr, col, keys


def _build(kind: str, scale_or_n: int, edge_factor_or_m: int, seed: int, probs, permute: bool,
           transpose: bool, backend: str, device):
    """Generate raw edges in chunks, relabel, dedup and return sorted unique keys."""
    if kind == "rmat":
        n = 1 << scale_or_n
        m_raw = n * edge_factor_or_m
    else:
        n = scale_or_n
        m_raw = edge_factor_or_m
    perm = random_permutation(n, seed, backend, device) if permute else None
    if backend == "np":
        keys = np.empty(m_raw, dtype=np.int64)
    else:
        import torch
        keys = torch.empty(m_raw, dtype=torch.int64, device=device)
    for start in range(0, m_raw, CHUNK):
        cnt = min(CHUNK, m_raw - start)
        if kind == "rmat":
            a, b, c = probs
            s, d = rmat_edges(scale_or_n, seed, a, b, c, start, cnt, backend, device)
        else:
            s, d = er_edges(n, seed, start, cnt, backend, device)
        if perm is not None:
            s, d = perm[s], perm[d]
        if transpose:
            s, d = d, s
        keys[start:start + cnt] = (s << 32) | d
        del s, d
    return n, m_raw, keys


CONFIGS = {
    # BASELINE.json configs[0..4]; "bits" = log2 partition size q.
    "c1": dict(name="c1_rmat10", kind="rmat", scale=10, edge_factor=16, seed=1,
               probs=(0.57, 0.19, 0.19), permute=False, bits=8, iters=10, op="pagerank"),
    "c2": dict(name="c2_er20", kind="er", n=1 << 20, m_raw=1 << 24, seed=2,
               permute=False, bits=15, iters=20, op="pagerank"),
    "c3": dict(name="c3_rmat24", kind="rmat", scale=24, edge_factor=16, seed=3,
               probs=(0.57, 0.19, 0.19), permute=True, bits=15, iters=20, op="pagerank"),
    "c4": dict(name="c4_rmat26", kind="rmat", scale=26, edge_factor=16, seed=4,
               probs=(0.57, 0.19, 0.19), permute=True, bits=15, iters=20, op="pagerank"),
    # configs[3] run twice: C4's graph relabelled by BFS order (reading R16)
    "c4bfs": dict(name="c4_rmat26_bfs", kind="rmat", scale=26, edge_factor=16, seed=4,
                  probs=(0.57, 0.19, 0.19), permute=True, bfs=True, bits=15, iters=20, op="pagerank"),
    "c5": dict(name="c5_spmv_rmat25", kind="rmat", scale=25, edge_factor=16, seed=5,
               probs=(0.57, 0.19, 0.19), permute=True, bits=15, iters=50, op="spmv"),
    # SURVEY §8(f)#4 benchmark lines (not BASELINE configs): weighted PageRank (P:287-288,
    # reading R24) on C4's graph with weights |U[-1,1)| keyed by the raw edge (R18), and a
    # non-square SpMV: C5's matrix restricted to its first half of the columns
    # (y = M^T x with M 2^25 x 2^24, "rows and columns partitioned separately")
    "c4w": dict(name="c4w_rmat26_weighted", kind="rmat", scale=26, edge_factor=16, seed=4,
                probs=(0.57, 0.19, 0.19), permute=True, bits=15, iters=20, op="pagerank", weights="abs"),
    "c5ns": dict(name="c5ns_spmv_rmat25_2to1", kind="rmat", scale=25, edge_factor=16, seed=5,
                 probs=(0.57, 0.19, 0.19), permute=True, bits=15, iters=50, op="spmv", cols_div=2),
}


def make_graph(kind: str, seed: int, *, scale: int = 0, edge_factor: int = 16, n: int = 0,
               m_raw: int = 0, probs=(0.57, 0.19, 0.19), permute: bool = False,
               values: bool = False, transpose: bool = False, backend: str = "np", device=None,
               name: str = "") -> GraphCSR:
    """Generic seeded graph -> canonical CSR (dedup, self-loops kept).

    With ``transpose`` the CSR rows are the raw edges' destinations, i.e. the
    CSR of A^T for the raw adjacency A (used by the SpMV config so that
    y = A x is computed as y = M^T x with M = A^T, reading R17).
    ``values`` draws float32 entries uniform in [-1, 1) keyed by the raw
    (i, j) entry of A, independent of storage order (R18).
    """
    if kind == "rmat":
        nn, m_raw_, keys = _build("rmat", scale, edge_factor, seed, probs, permute, transpose,
                                  backend, device)
    else:
        nn, m_raw_, keys = _build("er", n, m_raw, seed, None, permute, transpose, backend, device)
    row_ptr, col, ukeys = edges_to_csr(keys, nn, nn, backend)
    del keys
    vals = None
    if values:
        # raw entry (i, j) of A: key_A = i << 32 | j.  Stored key is (j << 32 | i) when transposed.
        if backend == "np":
            k = ukeys
            ka = ((k & 0xFFFFFFFF) << 32) | (k >> 32) if transpose else k
            vals = unit_values_np(seed, S_VAL, ka.astype(np.uint64))
        else:
            k = ukeys
            ka = ((k & 0xFFFFFFFF) << 32) | (k >> 32) if transpose else k
            vals = unit_values_torch(seed, S_VAL, ka)
    del ukeys
    meta = dict(m_raw=m_raw_, kind=kind, seed=seed, permute=permute, transpose=transpose)
    return GraphCSR(name or f"{kind}", nn, nn, row_ptr, col, vals, meta)


def column_prefix(g: GraphCSR, n_cols: int) -> GraphCSR:
    """The sub-matrix of g's columns [0, n_cols) (a non-square CSR, rows kept)."""
    keep = g.col < n_cols if g.backend == "np" else g.col.view(-1) < n_cols
    if g.backend == "np":
        cm = np.concatenate([np.zeros(1, np.int64), np.cumsum(keep, dtype=np.int64)])
    else:
        import torch
        cm = torch.cat([torch.zeros(1, dtype=torch.int64, device=g.col.device),
                        torch.cumsum(keep.to(torch.int64), 0)])
    rp = cm[g.row_ptr]
    vals = None if g.values is None else g.values[keep]
    return GraphCSR(g.name, g.n_src, n_cols, rp, g.col[keep], vals, dict(g.meta))


def make_x(n: int, seed: int, backend: str = "np", device=None):
    """SpMV input vector x[i] = 2 U(seed, 401, i) - 1 (float32, R18)."""
    if backend == "np":
        return unit_values_np(seed, S_X, np.arange(n, dtype=np.uint64))
    import torch
    return unit_values_torch(seed, S_X, torch.arange(n, dtype=torch.int64, device=device))


_BFS_LIB = None


def _bfs_lib():
    """inputs/bfs_order.c compiled with gcc on first use (input generation, not the method)."""
    global _BFS_LIB
    if _BFS_LIB is None:
        import ctypes
        import os
        import subprocess
        here = os.path.dirname(os.path.abspath(__file__))
        src, lib = os.path.join(here, "bfs_order.c"), os.path.join(here, "libinputs.so")
        if not os.path.exists(lib) or os.path.getmtime(lib) < os.path.getmtime(src):
            tmp = lib + f".tmp{os.getpid()}"
            subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-std=c11", "-o", tmp, src])
            os.replace(tmp, lib)
        _BFS_LIB = ctypes.CDLL(lib)
        P = ctypes.c_void_p
        _BFS_LIB.inputs_bfs_order.argtypes = [ctypes.c_int64, P, P, P]
        _BFS_LIB.inputs_bfs_order.restype = ctypes.c_int
    return _BFS_LIB


def bfs_order(n: int, row_ptr: np.ndarray, col: np.ndarray) -> np.ndarray:
    """new_id[v] for the BFS locality labelling of reading R16 (host, O(n + m))."""
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    cl = np.ascontiguousarray(col, dtype=np.uint32)
    out = np.empty(n, dtype=np.int64)
    rc = _bfs_lib().inputs_bfs_order(n, rp.ctypes.data, cl.ctypes.data, out.ctypes.data)
    if rc != 0:
        raise MemoryError("bfs_order")
    return out


def relabel(g: GraphCSR, new_id, name: str = "") -> GraphCSR:
    """CSR of the same graph with vertex v renamed new_id[v] (rows re-sorted)."""
    n = g.n_src
    if g.backend == "np":
        rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(g.row_ptr))
        keys = (new_id[rows] << 32) | new_id[g.col.astype(np.int64)]
        del rows
    else:
        import torch
        nid = torch.as_tensor(new_id, device=g.row_ptr.device)
        rows = torch.repeat_interleave(torch.arange(n, dtype=torch.int64, device=nid.device),
                                       g.row_ptr[1:] - g.row_ptr[:-1])
        keys = (nid[rows] << 32) | nid[g.col.to(torch.int64) & 0xFFFFFFFF]
        del rows, nid
    row_ptr, col, _ = edges_to_csr(keys, n, n, g.backend)
    return GraphCSR(name or g.name, n, n, row_ptr, col, None, dict(g.meta))


def make_config(key: str, backend: str = "np", device=None) -> GraphCSR:
    """Build BASELINE.json config ``key`` ('c1'..'c5', 'c4bfs')."""
    cfg = CONFIGS[key]
    if cfg["kind"] == "rmat":
        g = make_graph("rmat", cfg["seed"], scale=cfg["scale"], edge_factor=cfg["edge_factor"],
                       probs=cfg["probs"], permute=cfg["permute"],
                       values=cfg["op"] == "spmv" or "weights" in cfg,
                       transpose=cfg["op"] == "spmv", backend=backend, device=device, name=cfg["name"])
        if cfg.get("weights") == "abs":              # non-negative edge weights (R24)
            g.values = abs(g.values)
        if cfg.get("cols_div"):
            g = column_prefix(g, g.n_dst // cfg["cols_div"])
    else:
        g = make_graph("er", cfg["seed"], n=cfg["n"], m_raw=cfg["m_raw"], permute=cfg["permute"],
                       backend=backend, device=device, name=cfg["name"])
    if cfg.get("bfs"):
        h = g.to_numpy()
        new_id = bfs_order(g.n_src, h.row_ptr, h.col)
        del h
        g = relabel(g, new_id, cfg["name"])
    g.meta.update(cfg)
    return g
