"""Counter-based 64-bit generator, identical in numpy (uint64) and torch (int64).

h(seed, stream, i) = mix64( base(seed, stream) + (i + 1) * G )
base(seed, stream) = mix64( seed * G + stream * H )
mix64 = the splitmix64 finaliser (xor-shift / multiply, all mod 2^64),
G = 0x9E3779B97F4A7C15, H = 0xD1B54A32D192ED03.

Every draw is a pure function of (seed, stream, i), so the same edge or value
comes out whatever the chunking, device or thread count.
torch has no full uint64 arithmetic, so the torch version works on int64 with
wrapping multiplies and emulates logical right shifts with a mask.
"""
from __future__ import annotations

import numpy as np

G = 0x9E3779B97F4A7C15
H = 0xD1B54A32D192ED03
M1 = 0xBF58476D1CE4E5B9
M2 = 0x94D049BB133111EB
MASK64 = (1 << 64) - 1


def _mix64_int(z: int) -> int:
    z &= MASK64
    z = ((z ^ (z >> 30)) * M1) & MASK64
    z = ((z ^ (z >> 27)) * M2) & MASK64
    return z ^ (z >> 31)


def stream_base(seed: int, stream: int) -> int:
    """base(seed, stream) as a Python int in [0, 2^64)."""
    return _mix64_int((seed * G + stream * H) & MASK64)


def _mix64_np(z: np.ndarray) -> np.ndarray:
    z = z ^ (z >> np.uint64(30))
    z = z * np.uint64(M1)
    z = z ^ (z >> np.uint64(27))
    z = z * np.uint64(M2)
    return z ^ (z >> np.uint64(31))


def counter_hash_np(seed: int, stream: int, idx: np.ndarray) -> np.ndarray:
    """uint64 hashes h(seed, stream, idx) for an integer index array."""
    idx = np.asarray(idx, dtype=np.uint64)
    base = np.uint64(stream_base(seed, stream))
    with np.errstate(over="ignore"):
        z = base + (idx + np.uint64(1)) * np.uint64(G)
        return _mix64_np(z)


def _signed(c: int) -> int:
    c &= MASK64
    return c - (1 << 64) if c >= (1 << 63) else c


def _lsr(z, s: int):
    """Logical right shift of an int64 torch tensor."""
    return (z >> s) & ((1 << (64 - s)) - 1)


def counter_hash_torch(seed: int, stream: int, idx):
    """Same hashes as counter_hash_np, as an int64 torch tensor (bit pattern of the uint64)."""
    import torch
    idx = idx.to(torch.int64)
    base = _signed(stream_base(seed, stream))
    z = (idx + 1) * _signed(G) + base
    z = z ^ _lsr(z, 30)
    z = z * _signed(M1)
    z = z ^ _lsr(z, 27)
    z = z * _signed(M2)
    return z ^ _lsr(z, 31)


def u53_np(h: np.ndarray) -> np.ndarray:
    """Top 53 bits of the hash as an integer in [0, 2^53)."""
    return (h >> np.uint64(11)).astype(np.int64)


def u53_torch(h):
    return _lsr(h, 11)


def top_bits_np(h: np.ndarray, bits: int) -> np.ndarray:
    return (h >> np.uint64(64 - bits)).astype(np.int64)


def top_bits_torch(h, bits: int):
    return _lsr(h, 64 - bits)
