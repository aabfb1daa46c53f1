"""Counter-based PRNG (splitmix64) used for every synthetic tensor.

Recipe (frozen in DESIGN.md "Input recipe"):
    key   = (seed XOR (tensor_id * 0x9E3779B97F4A7C15)) + index      (mod 2^64)
    x     = splitmix64(key)
    value = lo + (x >> (64 - b))        for a range [lo, lo + 2^b)

The data seed is 230716273 (the arXiv id).  The Fiat-Shamir seed of a named
configuration is SHA256("zkdl-b200/fs-seed/" || name).
"""
from __future__ import annotations

import hashlib

import numpy as np

DATA_SEED = 230716273
_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def fs_seed(config_name: str) -> bytes:
    """32-byte Fiat-Shamir seed of a named configuration."""
    return hashlib.sha256(b"zkdl-b200/fs-seed/" + config_name.encode()).digest()


def splitmix64(z: np.ndarray) -> np.ndarray:
    z = z.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        z += _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return z


def _keys(seed: int, tensor_id: int, n: int, offset: int = 0) -> np.ndarray:
    base = (seed ^ ((tensor_id * 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF)) & 0xFFFFFFFFFFFFFFFF
    idx = np.arange(offset, offset + n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return idx + np.uint64(base)


def uniform_bits(seed: int, tensor_id: int, n: int, lo: int, bits: int, offset: int = 0) -> np.ndarray:
    """n int64 values uniform in [lo, lo + 2^bits), 1 <= bits <= 63."""
    if not 1 <= bits <= 63:
        raise ValueError("bits must be in [1, 63]")
    x = splitmix64(_keys(seed, tensor_id, n, offset))
    return (x >> np.uint64(64 - bits)).astype(np.int64) + np.int64(lo)


def uniform_range(seed: int, tensor_id: int, shape, lo: int, hi: int, dtype=np.int32) -> np.ndarray:
    """Tensor of the given shape, uniform in [lo, hi) where hi - lo is a power of two."""
    span = hi - lo
    bits = span.bit_length() - 1
    if span <= 0 or (1 << bits) != span:
        raise ValueError("hi - lo must be a positive power of two")
    n = int(np.prod(shape)) if len(shape) else 1
    if bits == 0:
        return np.full(shape, lo, dtype=dtype)
    return uniform_bits(seed, tensor_id, n, lo, bits).astype(dtype).reshape(shape)


# ---------------------------------------------------------------- the same generator on a torch device
def _lsr(z, k: int):
    """Logical right shift of int64 tensors holding uint64 bit patterns."""
    import torch
    return (z >> k) & ((1 << (64 - k)) - 1)


def _i64(u: int) -> int:
    """uint64 constant -> the int64 with the same bits (torch integer arithmetic wraps mod 2^64)."""
    u &= 0xFFFFFFFFFFFFFFFF
    return u - (1 << 64) if u >> 63 else u


def uniform_range_torch(seed: int, tensor_id: int, n: int, lo: int, hi: int, device, offset: int = 0,
                        chunk: int = 1 << 26):
    """int32 tensor of entries offset .. offset+n-1 of uniform_range(seed, tensor_id, ...) computed on
    `device` (bit-identical to the numpy generator; used for inputs too large to generate on the host,
    e.g. C5 at m = 30, and for per-rank slices of a sharded statement)."""
    import torch
    span = hi - lo
    bits = span.bit_length() - 1
    if span <= 0 or (1 << bits) != span or not 1 <= bits <= 63:
        raise ValueError("hi - lo must be a power of two in [2, 2^63]")
    base = (seed ^ ((tensor_id * 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF)) & 0xFFFFFFFFFFFFFFFF
    out = torch.empty(n, dtype=torch.int32, device=device)
    g, m1, m2 = _i64(0x9E3779B97F4A7C15), _i64(0xBF58476D1CE4E5B9), _i64(0x94D049BB133111EB)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        z = torch.arange(offset + s, offset + e, dtype=torch.int64, device=device) + _i64(base)
        z = z + g
        z = (z ^ _lsr(z, 30)) * m1
        z = (z ^ _lsr(z, 27)) * m2
        z = z ^ _lsr(z, 31)
        out[s:e] = (_lsr(z, 64 - bits) + lo).to(torch.int32)
    return out
