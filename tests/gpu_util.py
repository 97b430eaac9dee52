"""Test helpers for the GPU parity tests: device->host copies of exported layout
pointers (libcudart via ctypes) and CSR upload through torch."""
from __future__ import annotations

import ctypes
import os

import numpy as np

_cudart = None


def cudart():
    global _cudart
    if _cudart is None:
        import nvidia.cuda_runtime as cr
        base = list(cr.__path__)[0]
        _cudart = ctypes.CDLL(os.path.join(base, "lib", "libcudart.so.12"))
        _cudart.cudaMemcpy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
        _cudart.cudaMemcpy.restype = ctypes.c_int
    return _cudart


def d2h(ptr, count, dtype):
    """Copy `count` elements of `dtype` from device pointer `ptr` to a new numpy array."""
    out = np.zeros(max(int(count), 1), dtype=dtype)
    if count > 0:
        rc = cudart().cudaMemcpy(ctypes.c_void_p(out.ctypes.data), ctypes.c_void_p(ptr),
                                 int(count) * out.itemsize, 2)
        assert rc == 0, f"cudaMemcpy D2H failed ({rc})"
    return out[:int(count)]


def to_device(g):
    """(row_ptr, col, values) of a numpy GraphCSR as CUDA torch tensors."""
    import torch
    rp = torch.from_numpy(np.ascontiguousarray(g.row_ptr, dtype=np.int64)).cuda()
    col = torch.from_numpy(np.ascontiguousarray(g.col, dtype=np.uint32).view(np.int32)).cuda()
    val = None if g.values is None else torch.from_numpy(np.ascontiguousarray(g.values, dtype=np.float32)).cuda()
    return rp, col, val


def spmv_fbits(values, x):
    """Fractional bits F of the SpMV fixed-point accumulator, computed from the INPUTS
    as DESIGN.md R22 defines it (never read back from the library): F = 22 - e_w - e_x,
    e(a) = the exponent with max|a| < 2^e (frexp), e_w = 0 for a structure-only matrix
    (w = 1), clamped to [-120, 62].  Then every |w x| 2^F < 2^22."""
    import math
    ex = lambda a: math.frexp(float(np.max(np.abs(a))))[1] if len(a) and np.max(np.abs(a)) > 0 else 0  # noqa: E731
    vals = None if values is None else np.asarray(values, dtype=np.float32)
    f = 22 - (0 if vals is None else ex(vals)) - ex(np.asarray(x, dtype=np.float32))
    return max(-120, min(62, f))
