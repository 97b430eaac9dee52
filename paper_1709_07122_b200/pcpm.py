"""Thin ctypes binding of include/pcpm.h (argument marshalling only).

Every function has the C name and forwards to libpcpm.so; all computation runs
in the CUDA kernels of that library.  Arrays may be torch tensors (host or
CUDA) or numpy arrays (host); the library detects host vs device pointers.
If libpcpm.so is missing this module raises at import: there is no fallback.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PCPM_LIB") or os.path.join(_HERE, "libpcpm.so")   # PCPM_LIB: A/B variant builds

PCPM_OK = 0
PCPM_EINVAL = -1
PCPM_ETOOBIG = -2
PCPM_EBADCSR = -3
PCPM_ENOMEM = -4
PCPM_ECUDA = -5
PCPM_ESTATE = -6
PCPM_NO_COMPRESS = 0x1
PCPM_BUILD_PULL = 0x2
PCPM_KEEP_VALUES = 0x4
PCPM_WIDE_IDS = 0x8
PCPM_COMPACT_SLOTS = 0x10
PCPM_BVGAS = 0x20

EXPORTED = ["pcpm_build", "pcpm_build_ex", "pcpm_pagerank", "pcpm_spmv", "pcpm_pull_pagerank", "pcpm_destroy",
            "pcpm_set_stream", "pcpm_last_error", "pcpm_last_status", "pcpm_get_info", "pcpm_export_layout",
            "pcpm_get_residuals", "pcpm_scatter", "pcpm_set_option", "pcpm_last_launch_count",
            "pcpm_get_phase_times", "pcpm_build_shard", "pcpm_shard_init", "pcpm_shard_step", "pcpm_get_debug_counters",
            "pcpm_shard_step_peers", "pcpm_pagerank_tol", "pcpm_shard_init_peers", "pcpm_ipc_handle_bytes", "pcpm_ipc_alloc", "pcpm_ipc_free", "pcpm_ipc_get_handle",
            "pcpm_ipc_open", "pcpm_ipc_close", "pcpm_pool_reserve", "pcpm_runtime_create", "pcpm_job_submit",
            "pcpm_job_wait", "pcpm_runtime_destroy"]


class PcpmError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"pcpm error {code}: {msg}")
        self.code = code


class pcpm_csr(ctypes.Structure):
    _fields_ = [("n_src", ctypes.c_int64), ("n_dst", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("row_ptr", ctypes.c_void_p), ("col_idx", ctypes.c_void_p), ("values", ctypes.c_void_p)]


class pcpm_info(ctypes.Structure):
    _fields_ = [("n_src", ctypes.c_int64), ("n_dst", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("partition_bits", ctypes.c_int32), ("q", ctypes.c_int64), ("k_src", ctypes.c_int64),
                ("k_dst", ctypes.c_int64), ("e_prime", ctypes.c_int64), ("r", ctypes.c_double),
                ("n_dangling", ctypes.c_int64), ("weighted", ctypes.c_int32), ("compressed", ctypes.c_int32),
                ("device_bytes", ctypes.c_int64), ("build_ms", ctypes.c_double),
                ("gather_items", ctypes.c_int64), ("scatter_items", ctypes.c_int64),
                ("fixed_point_bits", ctypes.c_int32), ("compact_slots", ctypes.c_int32),
                ("fused_iterations", ctypes.c_int32), ("bvgas", ctypes.c_int32)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class pcpm_layout_view(ctypes.Structure):
    _fields_ = [("ids", ctypes.c_void_p), ("w", ctypes.c_void_p), ("png_src", ctypes.c_void_p),
                ("png_off", ctypes.c_void_p), ("upd_off", ctypes.c_void_p), ("bin_id_start", ctypes.c_void_p),
                ("bin_upd_start", ctypes.c_void_p), ("chunk_base", ctypes.c_void_p),
                ("out_degree", ctypes.c_void_p), ("upd", ctypes.c_void_p), ("chunk_ids", ctypes.c_int64),
                ("ids16", ctypes.c_void_p), ("png_src16", ctypes.c_void_p), ("wide", ctypes.c_int32)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                          "(python -m paper_1709_07122_b200.build_ext). There is no CPU fallback.")
    lib = ctypes.CDLL(LIB_PATH)
    P, I, I64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
    sig = {
        "pcpm_build": (P, [ctypes.POINTER(pcpm_csr), I]),
        "pcpm_build_ex": (P, [ctypes.POINTER(pcpm_csr), I, ctypes.c_uint, P]),
        "pcpm_pagerank": (I, [P, ctypes.c_double, I, P]),
        "pcpm_pull_pagerank": (I, [P, ctypes.c_double, I, P]),
        "pcpm_spmv": (I, [P, P, P]),
        "pcpm_destroy": (None, [P]),
        "pcpm_set_stream": (I, [P, P]),
        "pcpm_last_error": (I, [ctypes.c_char_p, I]),
        "pcpm_last_status": (I, []),
        "pcpm_get_info": (I, [P, ctypes.POINTER(pcpm_info)]),
        "pcpm_export_layout": (I, [P, ctypes.POINTER(pcpm_layout_view)]),
        "pcpm_get_residuals": (I, [P, P, I]),
        "pcpm_scatter": (I, [P, P]),
        "pcpm_set_option": (I, [P, ctypes.c_char_p, I64]),
        "pcpm_last_launch_count": (I64, [P]),
        "pcpm_get_phase_times": (I, [P, P, I]),
        "pcpm_build_shard": (P, [ctypes.POINTER(pcpm_csr), I, I64, I64, ctypes.c_uint, P]),
        "pcpm_shard_init": (I, [P, P, P, P]),
        "pcpm_shard_step": (I, [P, ctypes.c_double, P, P, P, P, P, P]),
        "pcpm_get_debug_counters": (I, [P, I, I]),
        "pcpm_shard_step_peers": (I, [P, ctypes.c_double, P, P, P, P, ctypes.POINTER(P), I, P]),
        "pcpm_shard_init_peers": (I, [P, P, ctypes.POINTER(P), I, P]),
        "pcpm_ipc_handle_bytes": (I, []),
        "pcpm_pagerank_tol": (I, [P, ctypes.c_double, ctypes.c_double, I, P, ctypes.POINTER(I)]),
        "pcpm_ipc_alloc": (I, [I64, ctypes.POINTER(P)]),
        "pcpm_ipc_free": (I, [P]),
        "pcpm_ipc_get_handle": (I, [P, P]),
        "pcpm_ipc_open": (I, [P, ctypes.POINTER(P)]),
        "pcpm_ipc_close": (I, [P]),
        "pcpm_pool_reserve": (I, [I64]),
        "pcpm_runtime_create": (P, []),
        "pcpm_job_submit": (I, [P, ctypes.POINTER(pcpm_csr), I, ctypes.c_uint, ctypes.c_double, I, P,
                                ctypes.POINTER(I64)]),
        "pcpm_job_wait": (I, [P, I64]),
        "pcpm_runtime_destroy": (None, [P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


_lib = _load()


def _ptr(a):
    """Raw pointer of a torch tensor / numpy array (None -> NULL)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be contiguous")
        return ctypes.c_void_p(a.ctypes.data)
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return ctypes.c_void_p(a.data_ptr())
    if isinstance(a, int):
        return ctypes.c_void_p(a)
    raise TypeError(f"unsupported array type {type(a)}")


def _check(rc):
    if rc != PCPM_OK:
        raise PcpmError(rc, pcpm_last_error())
    return rc


def pcpm_last_error() -> str:
    n = _lib.pcpm_last_error(None, 0)
    buf = ctypes.create_string_buffer(n + 1)
    _lib.pcpm_last_error(buf, n + 1)
    return buf.value.decode(errors="replace")


def pcpm_last_status() -> int:
    return _lib.pcpm_last_status()


def make_csr(n_src, n_dst, row_ptr, col_idx, values=None, nnz=None):
    """pcpm_csr over caller-owned arrays (keep them alive for the pcpm_build call).
    ``nnz`` defaults to row_ptr[-1] (read from the array: pass it when row_ptr is a device
    buffer still being written on another stream)."""
    if nnz is None:
        nnz = int(row_ptr[-1]) if not hasattr(row_ptr, "data_ptr") else int(row_ptr[-1].item())
    return pcpm_csr(int(n_src), int(n_dst), nnz, _ptr(row_ptr), _ptr(col_idx), _ptr(values))


def pcpm_build(csr: pcpm_csr, partition_bits: int):
    h = _lib.pcpm_build(ctypes.byref(csr), int(partition_bits))
    if not h:
        raise PcpmError(pcpm_last_status(), pcpm_last_error())
    return h


def pcpm_build_ex(csr: pcpm_csr, partition_bits: int, flags: int = 0, stream=None):
    h = _lib.pcpm_build_ex(ctypes.byref(csr), int(partition_bits), int(flags), _stream(stream))
    if not h:
        raise PcpmError(pcpm_last_status(), pcpm_last_error())
    return h


def _stream(stream):
    if stream is None:
        return None
    if hasattr(stream, "cuda_stream"):
        return ctypes.c_void_p(stream.cuda_stream)
    return ctypes.c_void_p(int(stream))


def pcpm_pagerank(h, d: float, iters: int, out):
    return _check(_lib.pcpm_pagerank(h, float(d), int(iters), _ptr(out)))


def pcpm_pull_pagerank(h, d: float, iters: int, out):
    return _check(_lib.pcpm_pull_pagerank(h, float(d), int(iters), _ptr(out)))


def pcpm_spmv(h, x, y):
    return _check(_lib.pcpm_spmv(h, _ptr(x), _ptr(y)))


def pcpm_scatter(h, x):
    return _check(_lib.pcpm_scatter(h, _ptr(x)))


def pcpm_destroy(h):
    if h:
        _lib.pcpm_destroy(h)


def pcpm_pool_reserve(nbytes: int):
    return _check(_lib.pcpm_pool_reserve(int(nbytes)))


def pcpm_set_stream(h, stream):
    return _check(_lib.pcpm_set_stream(h, _stream(stream)))


def pcpm_set_option(h, key: str, value: int):
    return _check(_lib.pcpm_set_option(h, key.encode(), int(value)))


def pcpm_get_info(h) -> pcpm_info:
    info = pcpm_info()
    _check(_lib.pcpm_get_info(h, ctypes.byref(info)))
    return info


def pcpm_export_layout(h) -> pcpm_layout_view:
    v = pcpm_layout_view()
    _check(_lib.pcpm_export_layout(h, ctypes.byref(v)))
    return v


def pcpm_get_residuals(h, cap: int = 4096) -> np.ndarray:
    buf = np.zeros(cap, dtype=np.float64)
    n = _lib.pcpm_get_residuals(h, _ptr(buf), int(cap))
    if n < 0:
        _check(n)
    return buf[:n]


def pcpm_last_launch_count(h) -> int:
    return int(_lib.pcpm_last_launch_count(h))


def pcpm_get_phase_times(h, cap: int = 8192) -> np.ndarray:
    buf = np.zeros(cap, dtype=np.float32)
    n = _lib.pcpm_get_phase_times(h, _ptr(buf), int(cap))
    if n < 0:
        _check(n)
    return buf[:n]


def pcpm_build_shard(csr: pcpm_csr, partition_bits: int, v_lo: int, v_hi: int, flags: int = 0, stream=None):
    h = _lib.pcpm_build_shard(ctypes.byref(csr), int(partition_bits), int(v_lo), int(v_hi), int(flags),
                              _stream(stream))
    if not h:
        raise PcpmError(pcpm_last_status(), pcpm_last_error())
    return h


def pcpm_shard_init(h, pr0, spr0, dang0):
    return _check(_lib.pcpm_shard_init(h, _ptr(pr0), _ptr(spr0), _ptr(dang0)))


def pcpm_shard_step(h, d: float, spr_in, D_in, pr_old, pr_new, spr_out, red_out):
    return _check(_lib.pcpm_shard_step(h, float(d), _ptr(spr_in), _ptr(D_in), _ptr(pr_old), _ptr(pr_new),
                                       _ptr(spr_out), _ptr(red_out)))


PCPM_MAX_PEERS = 8


def pcpm_shard_step_peers(h, d: float, spr_in, D_in, pr_old, pr_new, spr_outs, red_out):
    """pcpm_shard_step with the exchange fused: spr_outs = [own chunk, peer chunks...]
    (device pointers or tensors)."""
    outs = (ctypes.c_void_p * len(spr_outs))(*[_ptr(o).value for o in spr_outs])
    return _check(_lib.pcpm_shard_step_peers(h, float(d), _ptr(spr_in), _ptr(D_in), _ptr(pr_old), _ptr(pr_new),
                                             outs, len(spr_outs), _ptr(red_out)))


def pcpm_shard_init_peers(h, pr0, spr_outs, dang0):
    outs = (ctypes.c_void_p * len(spr_outs))(*[_ptr(o).value for o in spr_outs])
    return _check(_lib.pcpm_shard_init_peers(h, _ptr(pr0), outs, len(spr_outs), _ptr(dang0)))


def pcpm_pagerank_tol(h, d: float, tol: float, max_iters: int, out) -> int:
    """PageRank until the L1 residual <= tol (or max_iters); returns the iteration count."""
    done = ctypes.c_int(0)
    _check(_lib.pcpm_pagerank_tol(h, float(d), float(tol), int(max_iters), _ptr(out), ctypes.byref(done)))
    return done.value


def pcpm_ipc_alloc(nbytes: int) -> int:
    """A zeroed cudaMalloc'ed exchange buffer (device pointer as int)."""
    p = ctypes.c_void_p()
    _check(_lib.pcpm_ipc_alloc(int(nbytes), ctypes.byref(p)))
    return p.value


def pcpm_ipc_free(ptr: int):
    return _check(_lib.pcpm_ipc_free(ctypes.c_void_p(ptr)))


def pcpm_ipc_get_handle(ptr: int) -> bytes:
    buf = ctypes.create_string_buffer(_lib.pcpm_ipc_handle_bytes())
    _check(_lib.pcpm_ipc_get_handle(ctypes.c_void_p(ptr), buf))
    return buf.raw


def pcpm_ipc_open(handle: bytes) -> int:
    p = ctypes.c_void_p()
    _check(_lib.pcpm_ipc_open(ctypes.create_string_buffer(handle, len(handle)), ctypes.byref(p)))
    return p.value


def pcpm_ipc_close(ptr: int):
    return _check(_lib.pcpm_ipc_close(ctypes.c_void_p(ptr)))


def pcpm_get_debug_counters(reset: bool = True) -> np.ndarray:
    buf = np.zeros(24, dtype=np.uint64)
    n = _lib.pcpm_get_debug_counters(_ptr(buf), 24, int(reset))
    if n < 0:
        _check(n)
    return buf[:n]


def pcpm_runtime_create():
    rt = _lib.pcpm_runtime_create()
    if not rt:
        raise PcpmError(pcpm_last_status(), pcpm_last_error())
    return rt


def pcpm_job_submit(rt, csr: pcpm_csr, partition_bits: int, flags: int, d: float, iters: int, out) -> int:
    """Queue one PageRank job (host or device CSR -> PR in out); returns its id at once."""
    jid = ctypes.c_int64()
    _check(_lib.pcpm_job_submit(rt, ctypes.byref(csr), int(partition_bits), int(flags), float(d), int(iters),
                                _ptr(out), ctypes.byref(jid)))
    return jid.value


def pcpm_job_wait(rt, job_id: int):
    return _check(_lib.pcpm_job_wait(rt, int(job_id)))


def pcpm_runtime_destroy(rt):
    if rt:
        _lib.pcpm_runtime_destroy(rt)
