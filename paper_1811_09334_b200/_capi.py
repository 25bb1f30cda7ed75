"""ctypes declarations of librqlp.so (include/rqlp.h).  Argument marshalling only."""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "librqlp.so")

_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64
_int = ctypes.c_int
_vp = ctypes.c_void_p
_sz = ctypes.c_size_t

# (name, restype, argtypes) -- mirrors include/rqlp.h
SIGNATURES = [
    ("rqlp_create", _int, [ctypes.POINTER(_vp), _int, _vp]),
    ("rqlp_create_dist", _int, [ctypes.POINTER(_vp), _int, _vp, _vp, _int, _int]),
    ("rqlp_get_unique_id", _int, [_vp]),
    ("rqlp_create_loopback", _int, [ctypes.POINTER(_vp), _int, _int, _vp]),
    ("rqlp_destroy", _int, [_vp]),
    ("rqlp_workspace_size", _int, [_vp, _int, _i64, _i64, _int, _int, _int, _int, _int, ctypes.POINTER(_sz)]),
    ("rqlp_set_workspace", _int, [_vp, _vp, _sz]),
    ("rqlp", _int, [_i64, _i64, _int, _int, _int, _vp, _i64, _u64, _vp, _vp, _vp]),
    ("rqlp_ex", _int, [_vp, _i64, _i64, _int, _int, _int, _vp, _i64, _u64, _vp, _i64, _vp, _i64, _vp, _i64,
                       _vp, _vp]),
    ("erqlp_ex", _int, [_vp, _i64, _i64, _int, _int, _int, _int, _vp, _i64, _u64, _vp, _i64, _vp, _i64,
                        ctypes.POINTER(_int), _vp, _i64, _vp]),
    ("brqlp_ex", _int, [_vp, _i64, _i64, _int, _int, _int, _int, _vp, _i64, _u64, _vp, _i64, _vp, _i64, _vp, _i64,
                        _vp, _vp]),
    ("rqlp_tqlp_ex", _int, [_vp, _i64, _i64, _int, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _vp]),
    ("rqlp_autorank_ex", _int, [_vp, _i64, _i64, _int, _int, _int, ctypes.c_double, _vp, _i64, _u64, _vp, _i64,
                                _vp, _i64, _vp, _i64, _vp, _vp, ctypes.POINTER(_int), ctypes.POINTER(ctypes.c_double)]),
    ("rqlp_factorize", _int, [_vp, _int, _i64, _i64, _int, _int, _int, _int, _int, _vp, _i64, _u64, _vp, _vp, _vp,
                              ctypes.POINTER(_int)]),
    ("rqlp_sync", _int, [_vp, ctypes.POINTER(ctypes.c_uint)]),
    ("rqlp_get_indicator", _int, [_vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]),
    ("rqlp_strerror", ctypes.c_char_p, [_int]),
    ("rqlp_omega", _int, [_vp, _i64, _i64, _u64, _vp, _i64]),
    ("rqlp_gemm_nn", _int, [_vp, _i64, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _i64]),
    ("rqlp_gemm_tn", _int, [_vp, _i64, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _int]),
    ("rqlp_orth", _int, [_vp, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _i64]),
    ("rqlp_cpqr", _int, [_vp, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _vp]),
    ("rqlp_qlp_tail", _int, [_vp, _i64, _i64, _vp, _i64, _int, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _vp,
                             ctypes.POINTER(_int)]),
    ("rqlp_residual_sq", _int, [_vp, _i64, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _vp]),
    ("rqlp_set_stage_outputs", _int, [_vp, _vp, _i64, _vp, _i64, _vp, _i64]),
    ("rqlp_set_power_stage_outputs", _int, [_vp, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _i64]),
    ("rqlp_set_timing", _int, [_vp, _int]),
    ("rqlp_get_timing", _int, [_vp, ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(ctypes.c_float), _int]),
    ("rqlp_launch_count", _i64, [_vp]),
    ("rqlp_careful_rerun_count", _i64, [_vp]),
]

_lib = None


def load(path: str = LIB_PATH):
    """Load librqlp.so.  Raises (never falls back) when the CUDA extension is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise RuntimeError(f"librqlp.so not built at {path}: run `python -m paper_1811_09334_b200.build` "
                               "(there is no CPU fallback)")
        lib = ctypes.CDLL(path)
        for name, res, args in SIGNATURES:
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib
