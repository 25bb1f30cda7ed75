"""CPU oracle for RQLP / ERQLP / BRQLP (arXiv:1811.09334) -- ctypes binding of oracle.c.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The product package
``paper_1811_09334_b200`` never imports it, and shares no code with it.

All arrays are numpy float64 in Fortran (column-major) order, matching the C side.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
CFLAGS = ["-O2", "-fno-fast-math", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared", "-std=gnu11"]


def build(force: bool = False) -> str:
    """Compile liboracle.so (plain C99 + OpenMP, no FMA contraction)."""
    src_m = max(os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "oracle.h")))
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < src_m:
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


_lib = None
_d = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)
_u64p = ctypes.POINTER(ctypes.c_uint64)
_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64
_int = ctypes.c_int


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        L = _lib
        L.orc_philox4x64_10.argtypes = [_u64p, _u64p, _u64p]
        L.orc_uniform.argtypes = [_u64]
        L.orc_uniform.restype = ctypes.c_double
        L.orc_ln.argtypes = [ctypes.c_double]
        L.orc_ln.restype = ctypes.c_double
        L.orc_sincos_2pi.argtypes = [_u64, _d, _d]
        L.orc_normal4.argtypes = [_u64, _u64, _u64, _d]
        L.orc_gaussian.argtypes = [_u64, _u64, _i64, _i64, _d, _i64]
        for f in (L.orc_gemm_nn, L.orc_gemm_tn, L.orc_gemm_nt):
            f.argtypes = [_i64, _i64, _i64, _d, _i64, _d, _i64, _d, _i64]
        L.orc_fro.argtypes = [_i64, _i64, _d, _i64]
        L.orc_fro.restype = ctypes.c_double
        L.orc_hqr.argtypes = [_i64, _i64, _d, _i64, _d, _i64, _d, _i64]
        L.orc_cpqr.argtypes = [_i64, _i64, _d, _i64, _d, _i64, _d, _i64, _i64p]
        L.orc_cpqr_partial.argtypes = [_i64, _i64, _i64, _d, _i64, _d, _i64, _d, _i64, _i64p]
        L.orc_tqlp.argtypes = [_i64, _i64, _i64, _d, _i64, _d, _i64, _d, _i64, _d, _i64, _i64p, _i64p]
        L.orc_svd_values.argtypes = [_i64, _i64, _d, _i64, _d]
        L.orc_qlp_tail.argtypes = [_i64, _i64, _d, _i64, _int, _d, _i64, _d, _i64, _d, _i64,
                                   _i64p, _i64p, ctypes.POINTER(_int)]
        L.orc_rqlp.argtypes = [_i64, _i64, _int, _int, _int, _int, _d, _i64, _u64,
                               _d, _i64, _d, _i64, _d, _i64, _i64p, _i64p, ctypes.POINTER(_int),
                               _d, _i64, _d, _i64]
        L.orc_brqlp.argtypes = [_i64, _i64, _int, _int, _int, _int, _d, _i64, _u64,
                                _d, _i64, _d, _i64, _d, _i64, _i64p, _i64p, _d, _i64]
        L.orc_autorank.argtypes = [_i64, _i64, _int, _int, _int, ctypes.c_double, _d, _i64, _u64, _d, _i64, _d,
                                   _i64, _d, _i64, _i64p, _i64p, ctypes.POINTER(_int), ctypes.POINTER(ctypes.c_double)]
        L.orc_residual.argtypes = [_i64, _i64, _i64, _d, _i64, _d, _i64, _d, _i64, _d, _i64]
        L.orc_residual.restype = ctypes.c_double
        L.orc_num_threads.restype = _int
        L.orc_set_num_threads.argtypes = [_int]
    return _lib


def _f(a):
    """Column-major float64 view (copy if needed)."""
    return np.asfortranarray(a, dtype=np.float64)


def _p(a):
    return a.ctypes.data_as(_d) if a is not None else None


def _ld(a):
    return max(1, a.shape[0]) if a is not None else 1


def num_threads() -> int:
    return lib().orc_num_threads()


def set_num_threads(n: int) -> None:
    """OpenMP thread count of the following oracle calls (bench.py's single-thread sample)."""
    lib().orc_set_num_threads(int(n))


# ---------------- RNG ----------------
def philox(counter, key):
    c = (ctypes.c_uint64 * 4)(*[int(x) & (2**64 - 1) for x in counter])
    k = (ctypes.c_uint64 * 2)(*[int(x) & (2**64 - 1) for x in key])
    o = (ctypes.c_uint64 * 4)()
    lib().orc_philox4x64_10(c, k, o)
    return [int(x) for x in o]


def uniform(x: int) -> float:
    return lib().orc_uniform(int(x))


def ln(u: float) -> float:
    return lib().orc_ln(float(u))


def sincos_2pi(x: int):
    s, c = ctypes.c_double(), ctypes.c_double()
    lib().orc_sincos_2pi(int(x), ctypes.byref(s), ctypes.byref(c))
    return s.value, c.value


def normal4(seed: int, stream: int, block: int):
    z = np.zeros(4)
    lib().orc_normal4(seed, stream, block, _p(z))
    return z


def gaussian(seed: int, stream: int, rows: int, cols: int) -> np.ndarray:
    M = np.zeros((rows, cols), order="F")
    lib().orc_gaussian(seed, stream, rows, cols, _p(M), _ld(M))
    return M


def omega(seed: int, n: int, l: int) -> np.ndarray:
    """Ω (n x l), stream 0 (Alg.1 l.1)."""
    return gaussian(seed, 0, n, l)


# ---------------- dense blocks ----------------
def gemm_nn(A, B):
    A, B = _f(A), _f(B)
    C = np.zeros((A.shape[0], B.shape[1]), order="F")
    lib().orc_gemm_nn(A.shape[0], B.shape[1], A.shape[1], _p(A), _ld(A), _p(B), _ld(B), _p(C), _ld(C))
    return C


def gemm_tn(A, B):
    A, B = _f(A), _f(B)
    C = np.zeros((A.shape[1], B.shape[1]), order="F")
    lib().orc_gemm_tn(A.shape[1], B.shape[1], A.shape[0], _p(A), _ld(A), _p(B), _ld(B), _p(C), _ld(C))
    return C


def hqr(A):
    A = _f(A)
    m, n = A.shape
    Q = np.zeros((m, n), order="F")
    R = np.zeros((n, n), order="F")
    rc = lib().orc_hqr(m, n, _p(A), _ld(A), _p(Q), _ld(Q), _p(R), _ld(R))
    if rc != 0:
        raise ValueError(f"orc_hqr rc={rc}")
    return Q, R


def cpqr(A):
    A = _f(A)
    m, n = A.shape
    s = min(m, n)
    Q = np.zeros((m, s), order="F")
    R = np.zeros((s, n), order="F")
    perm = np.zeros(n, dtype=np.int64)
    rc = lib().orc_cpqr(m, n, _p(A), _ld(A), _p(Q), _ld(Q), _p(R), _ld(R), perm.ctypes.data_as(_i64p))
    if rc != 0:
        raise ValueError(f"orc_cpqr rc={rc}")
    return Q, R, perm


def cpqr_partial(A, k: int):
    """First k steps of the pivoted Householder QR: Q (m x k), R (k x n, pivot order), perm."""
    A = _f(A)
    m, n = A.shape
    Q = np.zeros((m, k), order="F")
    R = np.zeros((k, n), order="F")
    perm = np.zeros(n, dtype=np.int64)
    rc = lib().orc_cpqr_partial(m, n, k, _p(A), _ld(A), _p(Q), _ld(Q), _p(R), _ld(R), perm.ctypes.data_as(_i64p))
    if rc != 0:
        raise ValueError(f"orc_cpqr_partial rc={rc}")
    return Q, R, perm


def tqlp(A, l: int):
    """Truncated pivoted QLP (NEXT-3): dict(Q, T, P, piv0, piv1)."""
    A = _f(A)
    m, n = A.shape
    Q = np.zeros((m, l), order="F")
    L = np.zeros((l, l), order="F")
    P = np.zeros((n, l), order="F")
    piv0 = np.zeros(l, dtype=np.int64)
    piv1 = np.zeros(l, dtype=np.int64)
    rc = lib().orc_tqlp(m, n, l, _p(A), _ld(A), _p(Q), _ld(Q), _p(L), _ld(L), _p(P), _ld(P),
                        piv0.ctypes.data_as(_i64p), piv1.ctypes.data_as(_i64p))
    if rc != 0:
        raise ValueError(f"orc_tqlp rc={rc}")
    return dict(Q=Q, T=L, P=P, piv0=piv0, piv1=piv1)


def svd_values(A):
    A = _f(A)
    m, n = A.shape
    s = np.zeros(min(m, n))
    lib().orc_svd_values(m, n, _p(A), _ld(A), _p(s))
    return s


def fro(A):
    A = _f(A)
    return lib().orc_fro(A.shape[0], A.shape[1], _p(A), _ld(A))


# ---------------- the method ----------------
def qlp_tail(B, d: int = 0):
    B = _f(B)
    l, n = B.shape
    QB = np.zeros((l, l), order="F")
    T = np.zeros((l, l), order="F")
    PB = np.zeros((n, l), order="F")
    piv0 = np.zeros(l, dtype=np.int64)
    piv1 = np.zeros(l, dtype=np.int64)
    tu = ctypes.c_int(0)
    rc = lib().orc_qlp_tail(l, n, _p(B), _ld(B), d, _p(QB), l, _p(T), l, _p(PB), n,
                            piv0.ctypes.data_as(_i64p), piv1.ctypes.data_as(_i64p), ctypes.byref(tu))
    if rc != 0:
        raise ValueError(f"orc_qlp_tail rc={rc}")
    return dict(QB=QB, T=T, PB=PB, piv0=piv0, piv1=piv1, t_is_upper=bool(tu.value))


def rqlp(A, k: int, p: int, q: int = 0, d: int = 0, seed: int = 0, stages: bool = False):
    """RQLP (d=0, Alg. 1) / ERQLP (d>=1, Alg. 2) with q subspace iterations."""
    A = _f(A)
    m, n = A.shape
    l = k + p
    Q = np.zeros((m, l), order="F")
    T = np.zeros((l, l), order="F")
    P = np.zeros((n, l), order="F")
    piv0 = np.zeros(l, dtype=np.int64)
    piv1 = np.zeros(l, dtype=np.int64)
    tu = ctypes.c_int(0)
    V = np.zeros((m, l), order="F") if stages else None
    B = np.zeros((l, n), order="F") if stages else None
    rc = lib().orc_rqlp(m, n, k, p, q, d, _p(A), _ld(A), seed, _p(Q), _ld(Q), _p(T), _ld(T), _p(P), _ld(P),
                        piv0.ctypes.data_as(_i64p), piv1.ctypes.data_as(_i64p), ctypes.byref(tu),
                        _p(V), _ld(V), _p(B), _ld(B))
    if rc != 0:
        raise ValueError(f"orc_rqlp rc={rc}")
    out = dict(Q=Q, T=T, P=P, piv0=piv0, piv1=piv1, t_is_upper=bool(tu.value))
    if stages:
        out.update(V=V, B=B)
    return out


def brqlp(A, k: int, p: int, b: int, q: int = 0, seed: int = 0, stages: bool = False):
    """BRQLP (Alg. 3) with explicit deflation on a working copy, ragged last block."""
    A = _f(A)
    m, n = A.shape
    l = k + p
    Q = np.zeros((m, l), order="F")
    L = np.zeros((l, l), order="F")
    P = np.zeros((n, l), order="F")
    piv0 = np.zeros(l, dtype=np.int64)
    piv1 = np.zeros(l, dtype=np.int64)
    V = np.zeros((m, l), order="F") if stages else None
    rc = lib().orc_brqlp(m, n, k, p, b, q, _p(A), _ld(A), seed, _p(Q), _ld(Q), _p(L), _ld(L), _p(P), _ld(P),
                         piv0.ctypes.data_as(_i64p), piv1.ctypes.data_as(_i64p), _p(V), _ld(V))
    if rc != 0:
        raise ValueError(f"orc_brqlp rc={rc}")
    out = dict(Q=Q, T=L, P=P, piv0=piv0, piv1=piv1, t_is_upper=False)
    if stages:
        out.update(V=V)
    return out


def autorank(A, b: int, l_max: int, eps: float, q: int = 0, seed: int = 0):
    """Auto-rank RQLP (NEXT-1): blocks of b columns until ||A||^2 - sum ||B_j||^2 <= (eps ||A||)^2."""
    A = _f(A)
    m, n = A.shape
    Q = np.zeros((m, l_max), order="F")
    L = np.zeros((l_max, l_max), order="F")
    P = np.zeros((n, l_max), order="F")
    piv0 = np.zeros(l_max, dtype=np.int64)
    piv1 = np.zeros(l_max, dtype=np.int64)
    lo = ctypes.c_int(0)
    err = ctypes.c_double(0.0)
    rc = lib().orc_autorank(m, n, b, l_max, q, eps, _p(A), _ld(A), seed, _p(Q), _ld(Q), _p(L), _ld(L), _p(P), _ld(P),
                            piv0.ctypes.data_as(_i64p), piv1.ctypes.data_as(_i64p), ctypes.byref(lo),
                            ctypes.byref(err))
    if rc != 0:
        raise ValueError(f"orc_autorank rc={rc}")
    l = lo.value
    return dict(Q=Q[:, :l], T=L[:l, :l], P=P[:, :l], piv0=piv0[:l], piv1=piv1[:l], l=l, err=err.value)


def residual(A, Q, T, P) -> float:
    A, Q, T, P = _f(A), _f(Q), _f(T), _f(P)
    m, n = A.shape
    l = Q.shape[1]
    return lib().orc_residual(m, n, l, _p(A), _ld(A), _p(Q), _ld(Q), _p(T), _ld(T), _p(P), _ld(P))
