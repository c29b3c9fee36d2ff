"""Seeded counter-based synthetic input generator (host side).

Holds none of the method's arithmetic -- it only draws the paper's workload
(PAPER.md P:317-323): x in {+1,-1}^N (int8) or N(0,1) (fp32), a planted
uniform shift k0 and t = the K-window of x at k0 with bit flips (int8) or
Gaussian noise (fp32).  See tmgen.c for the exact definition; the device
generator ``tm_generate`` re-implements it bit-for-bit for integer outputs.
Used by tests, smoke() and bench.py to build inputs for both the oracle and
the GPU path.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "tmgen.c")
_LIB = os.path.join(_HERE, "libtmgen.so")
_u64, _i64, _p, _d = ctypes.c_uint64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_double

TAG_K0 = 0x4000000000000000
TAG_FLIP = 0x5000000000000000
TAG_TNOISE = 0x6000000000000000


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared",
                               "-ffp-contract=off", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        L.tg_key.restype = _u64
        L.tg_key.argtypes = [_u64, _u64]
        L.tg_hash.restype = _u64
        L.tg_hash.argtypes = [_u64, _u64, _u64]
        L.tg_gauss.restype = _d
        L.tg_gauss.argtypes = [_u64]
        L.tg_k0.restype = _i64
        L.tg_k0.argtypes = [_u64, _u64, _i64]
        L.tg_x_i8.restype = None
        L.tg_x_i8.argtypes = [_u64, _u64, _i64, _i64, _p]
        L.tg_x_f32.restype = None
        L.tg_x_f32.argtypes = [_u64, _u64, _i64, _i64, _p]
        L.tg_t_i8.restype = None
        L.tg_t_i8.argtypes = [_u64, _u64, _i64, _i64, _d, _p]
        L.tg_t_f32.restype = None
        L.tg_t_f32.argtypes = [_u64, _u64, _i64, _i64, _d, _p]
        L.tg_batch_i8.restype = None
        L.tg_batch_i8.argtypes = [_u64, _u64, _i64, _i64, _i64, _d, _p, _i64, _p, _p]
        L.tg_batch_f32.restype = None
        L.tg_batch_f32.argtypes = [_u64, _u64, _i64, _i64, _i64, _d, _p, _i64, _p, _p]
        _lib = L
    return _lib


def hash64(seed: int, pair: int, ctr: int) -> int:
    return lib().tg_hash(seed, pair, ctr)


def k0(seed: int, pair: int, N: int) -> int:
    return lib().tg_k0(seed, pair, N)


def signal(seed: int, pair: int, N: int, dtype=np.int8, lo: int = 0, length: int | None = None) -> np.ndarray:
    length = N - lo if length is None else length
    if np.dtype(dtype) == np.int8:
        out = np.empty(length, np.int8)
        lib().tg_x_i8(seed, pair, lo, length, out.ctypes.data)
    else:
        out = np.empty(length, np.float32)
        lib().tg_x_f32(seed, pair, lo, length, out.ctypes.data)
    return out


def template(seed: int, pair: int, N: int, K: int, noise: float = 0.0, dtype=np.int8) -> np.ndarray:
    """int8: noise = bit-flip probability; fp32: noise = Gaussian sigma."""
    if np.dtype(dtype) == np.int8:
        out = np.empty(K, np.int8)
        lib().tg_t_i8(seed, pair, N, K, noise, out.ctypes.data)
    else:
        out = np.empty(K, np.float32)
        lib().tg_t_f32(seed, pair, N, K, noise, out.ctypes.data)
    return out


def batch(seed: int, pair0: int, B: int, N: int, K: int, noise: float = 0.0, dtype=np.int8,
          x_out: np.ndarray | None = None, want_x: bool = True):
    """Return (x [B, N], t [B, K], k0 [B]) for pairs [pair0, pair0+B)."""
    dt = np.dtype(dtype)
    if want_x:
        x = x_out if x_out is not None else np.empty((B, N), dt)
        assert x.shape == (B, N) and x.dtype == dt and x.flags["C_CONTIGUOUS"]
        xp, ldx = x.ctypes.data, N
    else:
        x, xp, ldx = None, None, N
    t = np.empty((B, K), dt)
    k = np.empty(B, np.int64)
    fn = lib().tg_batch_i8 if dt == np.int8 else lib().tg_batch_f32
    fn(seed, pair0, B, N, K, noise, xp, ldx, t.ctypes.data, k.ctypes.data)
    return x, t, k
