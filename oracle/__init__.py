"""CPU oracle of Algorithm 1 (arXiv 1509.04863).

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may import this
package.  The product path (``paper_1509_04863_b200``) never imports it, and
this package never imports the product path.

The arithmetic lives in ``oracle.c`` (plain C, literal loops, int64 for int8
data and fp64 for fp32 data); this module only marshals numpy arrays through
ctypes.  Every function is pinned in ``tests/test_oracle.py``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

_i64 = ctypes.c_int64
_p = ctypes.c_void_p


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so with gcc (no fast-math: fp64 sums keep
    the literal left-to-right order of the paper's formulas)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared",
                               "-fno-fast-math", "-ffp-contract=off", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        L.or_ceil_div.restype = _i64
        L.or_ceil_div.argtypes = [_i64, _i64]
        L.or_moduli.restype = ctypes.c_int
        L.or_moduli.argtypes = [_i64, _i64, _i64, ctypes.POINTER(_i64), ctypes.POINTER(_i64)]
        for n in ("or_fold_i8", "or_fold_f32"):
            getattr(L, n).restype = None
            getattr(L, n).argtypes = [_p, _i64, _i64, _i64, _i64, _i64, _p]
        for n in ("or_correlate_i64", "or_correlate_f64"):
            getattr(L, n).restype = None
            getattr(L, n).argtypes = [_p, _i64, _i64, _p, _p]
        L.or_correlate_at_i64.restype = None
        L.or_correlate_at_i64.argtypes = [_p, _i64, _p, _p, _i64, _p]
        for n in ("or_argmax_i64", "or_argmax_f64"):
            getattr(L, n).restype = _i64
            getattr(L, n).argtypes = [_p, _i64]
        L.or_fold_bins_i8.restype = None
        L.or_fold_bins_i8.argtypes = [_p, _i64, _i64, _p, _i64, _p]
        L.or_crt.restype = _i64
        L.or_crt.argtypes = [_i64, _i64, _i64, _i64]
        L.or_crt_sets.restype = _i64
        L.or_crt_sets.argtypes = [_i64, _i64, _i64, _i64, _i64]
        L.or_crt_sets_modN.restype = _i64
        L.or_crt_sets_modN.argtypes = [_i64, _i64, _i64, _i64, _i64]
        L.or_resolve.restype = _i64
        L.or_resolve.argtypes = [_i64, _i64, _i64, _i64, _i64, ctypes.c_int]
        for n in ("or_ftm_i8", "or_ftm_f32"):
            getattr(L, n).restype = _i64
            getattr(L, n).argtypes = [_p, _i64, _p, _i64, _i64, ctypes.c_int, _p, _p, _p, _p, _p]
        for n in ("or_full_corr_i8", "or_full_corr_f32"):
            getattr(L, n).restype = None
            getattr(L, n).argtypes = [_p, _i64, _p, _i64, _p]
        L.or_phi_dense.restype = None
        L.or_phi_dense.argtypes = [_i64, _i64, _i64, _p]
        L.or_thm1_That_y_i64.restype = None
        L.or_thm1_That_y_i64.argtypes = [_p, _i64, _p, _i64, _p]
        for n in ("or_block_fold_i8", "or_block_fold_f32"):
            getattr(L, n).restype = None
            getattr(L, n).argtypes = [_p, _i64, _i64, _p, _p]
        L.or_block_correlate_f64.restype = None
        L.or_block_correlate_f64.argtypes = [_p, _i64, _p, _i64, _p]
        L.or_crt_multi.restype = _i64
        L.or_crt_multi.argtypes = [_p, _p, ctypes.c_int]
        L.or_crt_sets_multi.restype = _i64
        L.or_crt_sets_multi.argtypes = [_p, _p, ctypes.c_int, _i64]
        for n in ("or_ftm_multi_i8", "or_ftm_multi_f32"):
            getattr(L, n).restype = _i64
            getattr(L, n).argtypes = [_p, _i64, _p, _i64, _p, ctypes.c_int, _p]
        for n in ("or_ftm_block_i8", "or_ftm_block_f32"):
            getattr(L, n).restype = _i64
            getattr(L, n).argtypes = [_p, _i64, _p, _i64, _i64, _p, _p, _p, _p, _p]
        _lib = L
    return _lib


def _ptr(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


def _is_int(x: np.ndarray) -> bool:
    return x.dtype == np.int8


def _as_input(x: np.ndarray) -> np.ndarray:
    x = np.asarray(x)
    if x.dtype == np.int8:
        return np.ascontiguousarray(x)
    if x.dtype == np.float32:
        return np.ascontiguousarray(x)
    raise TypeError(f"oracle input must be int8 or float32, got {x.dtype}")


# --------------------------------------------------------------------------
# O1  Alg. 1 step 2
# --------------------------------------------------------------------------
def moduli(N: int, K: int, M: int = 0):
    """(M1, M2) = (M or K, M1+1); raises ValueError unless K <= M1 and M1*M2 > N."""
    a, b = _i64(), _i64()
    if lib().or_moduli(N, K, M, ctypes.byref(a), ctypes.byref(b)) != 0:
        raise ValueError(f"invalid (N={N}, K={K}, M={M}): need K <= M1 and M1*(M1+1) > N")
    return a.value, b.value


def ceil_div(a: int, b: int) -> int:
    return lib().or_ceil_div(a, b)


# --------------------------------------------------------------------------
# O2  Eq. (2) fold, Alg. 1 step 3, strategy 1
# --------------------------------------------------------------------------
def fold(x: np.ndarray, M: int, K: int, lo: int = 0, length: int | None = None) -> np.ndarray:
    """y[k] = sum_{i<ceil(N/M)} x[(k+iM) mod N], k < M+K; only positions in
    [lo, lo+length) contribute (the partial fold).  int8 -> int64, f32 -> f64."""
    x = _as_input(x)
    N = x.shape[0]
    length = N - lo if length is None else length
    assert 0 <= lo and lo + length <= N
    if _is_int(x):
        y = np.zeros(M + K, np.int64)
        lib().or_fold_i8(_ptr(x), N, M, K, lo, length, _ptr(y))
    else:
        y = np.zeros(M + K, np.float64)
        lib().or_fold_f32(_ptr(x), N, M, K, lo, length, _ptr(y))
    return y


def fold_bins(x: np.ndarray, M: int, bins) -> np.ndarray:
    """Selected entries y[k] of the Eq. (2) fold (int8 data), one by one."""
    x = _as_input(x)
    assert _is_int(x)
    bins = np.ascontiguousarray(np.asarray(bins, np.int64))
    out = np.zeros(bins.shape[0], np.int64)
    lib().or_fold_bins_i8(_ptr(x), x.shape[0], M, _ptr(bins), bins.shape[0], _ptr(out))
    return out


# --------------------------------------------------------------------------
# O3  correlation, Alg. 1 steps 4-6 read as P:61 (reading C3)
# --------------------------------------------------------------------------
def correlate(y: np.ndarray, M: int, t: np.ndarray) -> np.ndarray:
    """r[k] = sum_{i<K} t[i] y[k+i], k < M (direct; y has >= M+K-1 entries)."""
    t = _as_input(t)
    K = t.shape[0]
    assert y.shape[0] >= M + K - 1
    if _is_int(t):
        y = np.ascontiguousarray(y, np.int64)
        if y.shape[0] < M + K:
            y = np.concatenate([y, np.zeros(M + K - y.shape[0], np.int64)])
        r = np.zeros(M, np.int64)
        lib().or_correlate_i64(_ptr(y), M, K, _ptr(t), _ptr(r))
    else:
        y = np.ascontiguousarray(y, np.float64)
        if y.shape[0] < M + K:
            y = np.concatenate([y, np.zeros(M + K - y.shape[0], np.float64)])
        r = np.zeros(M, np.float64)
        lib().or_correlate_f64(_ptr(y), M, K, _ptr(t), _ptr(r))
    return r


def correlate_at(y: np.ndarray, t: np.ndarray, ks) -> np.ndarray:
    """r[k] = sum_{i<K} t[i] y[k+i] at the selected outputs ks only (int8 t, int64 y)."""
    t = _as_input(t)
    assert _is_int(t)
    y = np.ascontiguousarray(y, np.int64)
    ks = np.ascontiguousarray(np.asarray(ks, np.int64))
    assert ks.size == 0 or (ks.min() >= 0 and ks.max() + t.shape[0] <= y.shape[0])
    r = np.zeros(ks.shape[0], np.int64)
    lib().or_correlate_at_i64(_ptr(y), t.shape[0], _ptr(t), _ptr(ks), ks.shape[0], _ptr(r))
    return r


# --------------------------------------------------------------------------
# O4  Alg. 1 step 7, ties to the lowest index (reading C7)
# --------------------------------------------------------------------------
def argmax(r: np.ndarray) -> int:
    if r.dtype == np.int64:
        r = np.ascontiguousarray(r)
        return lib().or_argmax_i64(_ptr(r), r.shape[0])
    r = np.ascontiguousarray(r, np.float64)
    return lib().or_argmax_f64(_ptr(r), r.shape[0])


# --------------------------------------------------------------------------
# O5  Theorem 4 and Alg. 1 steps 8-9
# --------------------------------------------------------------------------
def crt(m1: int, M1: int, m2: int, M2: int) -> int:
    return lib().or_crt(m1, M1, m2, M2)


def crt_sets(m1: int, M1: int, m2: int, M2: int, N: int) -> int:
    return lib().or_crt_sets(m1, M1, m2, M2, N)


def crt_sets_modN(m1: int, M1: int, m2: int, M2: int, N: int) -> int:
    """Steps 8-9 with the candidate sets reduced mod N (reading C10's repair)."""
    return lib().or_crt_sets_modN(m1, M1, m2, M2, N)


def resolve(m1: int, M1: int, m2: int, M2: int, N: int, alias_repair: bool = False) -> int:
    return lib().or_resolve(m1, M1, m2, M2, N, int(alias_repair))


# --------------------------------------------------------------------------
# O6  Algorithm 1 end to end
# --------------------------------------------------------------------------
def ftm(x: np.ndarray, t: np.ndarray, M: int = 0, want_vectors: bool = True, alias_repair: bool = False) -> dict:
    """Run FTM() on one (signal, template) pair.  Returns a dict with k
    (-1 = NO_MATCH), residues, and (optionally) y1, y2, r1, r2.  alias_repair:
    steps 8-9 with the candidate sets reduced mod N (reading C10)."""
    x = _as_input(x)
    t = _as_input(t)
    N, K = x.shape[0], t.shape[0]
    M1, M2 = moduli(N, K, M)
    res = np.zeros(2, np.int64)
    if _is_int(x):
        assert _is_int(t)
        dt = np.int64
        fn = lib().or_ftm_i8
    else:
        assert t.dtype == np.float32
        dt = np.float64
        fn = lib().or_ftm_f32
    if want_vectors:
        y1 = np.zeros(M1 + K, dt); y2 = np.zeros(M2 + K, dt)
        r1 = np.zeros(M1, dt); r2 = np.zeros(M2, dt)
        k = fn(_ptr(x), N, _ptr(t), K, M, int(alias_repair), _ptr(res), _ptr(y1), _ptr(y2), _ptr(r1), _ptr(r2))
        return dict(k=k, residues=(int(res[0]), int(res[1])), M1=M1, M2=M2,
                    y1=y1, y2=y2, r1=r1, r2=r2)
    k = fn(_ptr(x), N, _ptr(t), K, M, int(alias_repair), _ptr(res), None, None, None, None)
    return dict(k=k, residues=(int(res[0]), int(res[1])), M1=M1, M2=M2)


# --------------------------------------------------------------------------
# Aux: brute force, dense Phi, Theorem 1's T^
# --------------------------------------------------------------------------
def full_corr(x: np.ndarray, t: np.ndarray) -> np.ndarray:
    """(Tx)_k = sum_{i<K} t_i x_{(k+i) mod N} for every k < N (N*K work)."""
    x = _as_input(x)
    t = _as_input(t)
    N, K = x.shape[0], t.shape[0]
    if _is_int(x):
        s = np.zeros(N, np.int64)
        lib().or_full_corr_i8(_ptr(x), N, _ptr(t), K, _ptr(s))
    else:
        s = np.zeros(N, np.float64)
        lib().or_full_corr_f32(_ptr(x), N, _ptr(t), K, _ptr(s))
    return s


def phi_dense(N: int, M: int, rows: int) -> np.ndarray:
    """D_rows(circ(r)) with r_k = 1 iff k mod M == 0 (Eq. 3), int8 [rows, N]."""
    P = np.zeros((rows, N), np.int8)
    lib().or_phi_dense(N, M, rows, _ptr(P))
    return P


def thm1_That_y(y: np.ndarray, M: int, t: np.ndarray) -> np.ndarray:
    """(T^ y)_i with T^ = circ([t 0_{M-K}]) on y[0..M) (Theorem 1)."""
    y = np.ascontiguousarray(y[:M], np.int64)
    t = _as_input(t)
    out = np.zeros(M, np.int64)
    lib().or_thm1_That_y_i64(_ptr(y), M, _ptr(t), t.shape[0], _ptr(out))
    return out


# --------------------------------------------------------------------------
# Strategy 2: the Block sampling matrix of Theorem 2
# --------------------------------------------------------------------------
def block_fold(x: np.ndarray, M: int, phi: np.ndarray | None = None) -> np.ndarray:
    """y = [Phi_M ... Phi_M] x_pad (x zero-padded to a multiple of M),
    Phi_M = circ(phi); phi None = Eq. (3)'s r on one block (Phi_M = I)."""
    x = _as_input(x)
    N = x.shape[0]
    if _is_int(x):
        y = np.zeros(M, np.int64)
        ph = None if phi is None else np.ascontiguousarray(phi, np.int8)
        lib().or_block_fold_i8(_ptr(x), N, M, None if ph is None else _ptr(ph), _ptr(y))
    else:
        y = np.zeros(M, np.float64)
        ph = None if phi is None else np.ascontiguousarray(phi, np.float32)
        lib().or_block_fold_f32(_ptr(x), N, M, None if ph is None else _ptr(ph), _ptr(y))
    return y


def block_correlate(y: np.ndarray, M: int, t: np.ndarray) -> np.ndarray:
    """(T^ y)_i, T^ = circ([t 0_{M-K}]) (Theorem 2): cyclic correlation."""
    t = _as_input(t)
    if _is_int(t):
        return thm1_That_y(np.ascontiguousarray(y, np.int64), M, t)
    y = np.ascontiguousarray(y[:M], np.float64)
    out = np.zeros(M, np.float64)
    lib().or_block_correlate_f64(_ptr(y), M, _ptr(t), t.shape[0], _ptr(out))
    return out


def ftm_block(x: np.ndarray, t: np.ndarray, M: int = 0, want_vectors: bool = True) -> dict:
    """FTM() with strategy 2 (Block Phi, Phi_M = I): y_j has M_j entries and
    the correlation is cyclic (T^ = circ(t)); steps 7-9 as in ftm()."""
    x = _as_input(x)
    t = _as_input(t)
    N, K = x.shape[0], t.shape[0]
    M1, M2 = moduli(N, K, M)
    res = np.zeros(2, np.int64)
    if _is_int(x):
        assert _is_int(t)
        dt, fn = np.int64, lib().or_ftm_block_i8
    else:
        assert t.dtype == np.float32
        dt, fn = np.float64, lib().or_ftm_block_f32
    if not want_vectors:
        k = fn(_ptr(x), N, _ptr(t), K, M, _ptr(res), None, None, None, None)
        return dict(k=k, residues=(int(res[0]), int(res[1])), M1=M1, M2=M2)
    y1 = np.zeros(M1, dt); y2 = np.zeros(M2, dt)
    r1 = np.zeros(M1, dt); r2 = np.zeros(M2, dt)
    k = fn(_ptr(x), N, _ptr(t), K, M, _ptr(res), _ptr(y1), _ptr(y2), _ptr(r1), _ptr(r2))
    return dict(k=k, residues=(int(res[0]), int(res[1])), M1=M1, M2=M2, y1=y1, y2=y2, r1=r1, r2=r2)


# --------------------------------------------------------------------------
# Theorem 4 with alpha moduli
# --------------------------------------------------------------------------
def crt_multi(m, M) -> int:
    """The unique z in [0, prod M) with z = m_j (mod M_j); -1 if not co-prime."""
    m = np.ascontiguousarray(m, np.int64); M = np.ascontiguousarray(M, np.int64)
    return lib().or_crt_multi(_ptr(m), _ptr(M), len(M))


def crt_sets_multi(m, M, N: int) -> int:
    """Steps 8-9 literally: the common element of the alpha candidate sets."""
    m = np.ascontiguousarray(m, np.int64); M = np.ascontiguousarray(M, np.int64)
    return lib().or_crt_sets_multi(_ptr(m), _ptr(M), len(M), N)


def ftm_multi(x: np.ndarray, t: np.ndarray, moduli) -> dict:
    """FTM() over alpha pairwise co-prime moduli (int8 or float32 data): k and residues."""
    x = _as_input(x); t = _as_input(t)
    M = np.ascontiguousarray(moduli, np.int64)
    res = np.zeros(len(M), np.int64)
    fn = lib().or_ftm_multi_i8 if _is_int(x) else lib().or_ftm_multi_f32
    k = fn(_ptr(x), x.shape[0], _ptr(t), t.shape[0], _ptr(M), len(M), _ptr(res))
    if k == -3:
        raise ValueError("moduli must be >= K, pairwise co-prime, with product > N")
    return dict(k=k, residues=tuple(int(v) for v in res))
