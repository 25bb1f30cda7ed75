"""CPU-only checks of the boundary: librqlp.so builds for sm_100a, loads, and exports every
symbol include/rqlp.h declares (no compute calls: there is no GPU here)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def libpath():
    from paper_1811_09334_b200 import build as rqbuild
    return rqbuild.build()


def header_symbols():
    src = open(os.path.join(ROOT, "include", "rqlp.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w]+\s*\*?\s*(\w+)\s*\(", src, flags=re.M)))


def test_header_declares_the_north_star_entry_points():
    syms = header_symbols()
    for s in ("rqlp", "rqlp_ex", "erqlp_ex", "brqlp_ex", "rqlp_create", "rqlp_create_dist", "rqlp_workspace_size"):
        assert s in syms


def test_library_exports_every_header_symbol(libpath):
    out = subprocess.check_output(["nm", "-D", "--defined-only", libpath], text=True)
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    missing = [s for s in header_symbols() if s not in exported]
    assert not missing, missing


def test_library_loads_and_binding_matches(libpath):
    lib = ctypes.CDLL(libpath)
    from paper_1811_09334_b200 import _capi
    for name, _, _ in _capi.SIGNATURES:
        assert hasattr(lib, name), name
    assert set(n for n, _, _ in _capi.SIGNATURES) == set(header_symbols())
    lib.rqlp_strerror.restype = ctypes.c_char_p
    assert lib.rqlp_strerror(0) == b"success"
    assert b"argument" in lib.rqlp_strerror(-3)


def test_sass_uses_dmma(libpath):
    """The FP64 GEMMs issue DMMA (the FP64 tensor pipe), not DFMA-only code."""
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "-sass", libpath], text=True)
    assert "DMMA.8x8x4" in out


def test_no_cpu_fallback_without_library(tmp_path):
    from paper_1811_09334_b200 import _capi
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _capi._lib = None
        try:
            _capi.load(str(tmp_path / "missing.so"))
        finally:
            _capi._lib = None


def test_argument_errors_without_gpu(libpath):
    """rqlp() validates arguments before touching the device (LAPACK-style -i codes)."""
    lib = ctypes.CDLL(libpath)
    i64, c_int, vp = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
    lib.rqlp.argtypes = [i64, i64, c_int, c_int, c_int, vp, i64, ctypes.c_uint64, vp, vp, vp]
    dummy = ctypes.c_void_p(1)
    assert lib.rqlp(0, 10, 3, 2, 0, dummy, 10, 0, dummy, dummy, dummy) == -1
    assert lib.rqlp(10, 10, 1, 2, 0, dummy, 10, 0, dummy, dummy, dummy) == -3
    assert lib.rqlp(10, 10, 3, 1, 0, dummy, 10, 0, dummy, dummy, dummy) == -4
    assert lib.rqlp(10, 10, 3, 2, -1, dummy, 10, 0, dummy, dummy, dummy) == -5
    assert lib.rqlp(10, 10, 3, 2, 0, None, 10, 0, dummy, dummy, dummy) == -6
    assert lib.rqlp(10, 10, 3, 2, 0, dummy, 9, 0, dummy, dummy, dummy) == -7
