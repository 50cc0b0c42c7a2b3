"""The C-ABI library loads on a CPU-only host and exports every symbol that
include/hh.h declares (no compute calls: those need a GPU)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hh.h")
LIB = os.path.join(ROOT, "paper_2104_01439_b200", "libhh.so")


def declared_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(hh_[a-z_0-9]+)\s*\(", txt)))


def test_header_declares_the_boundary_calls():
    syms = declared_symbols()
    for name in ("hh_setup_problem", "hh_apply_op", "hh_vcycle", "hh_fgmres_solve", "hh_sweep",
                 "hh_destroy_problem", "hh_last_error"):
        assert name in syms


def test_library_exports_every_declared_symbol():
    if not os.path.exists(LIB):
        import __graft_entry__
        __graft_entry__.build()
    import torch  # noqa: F401  (provides libcudart.so.12 to the loader)
    lib = ctypes.CDLL(LIB)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    lib.hh_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.hh_version()


def test_binding_exports_match_header():
    import paper_2104_01439_b200.hh as hh
    assert sorted(hh.EXPORTS) == declared_symbols()


def _lib():
    import torch  # noqa: F401
    return ctypes.CDLL(LIB)


class _Q(ctypes.Structure):   # hh_lfa_query
    _fields_ = [("k", ctypes.c_double), ("h", ctypes.c_double), ("beta", ctypes.c_double),
                ("sigma", ctypes.c_double), ("omega", ctypes.c_double), ("nu1", ctypes.c_int32),
                ("nu2", ctypes.c_int32), ("m", ctypes.c_int32), ("pad", ctypes.c_int32)]


def test_lfa_argument_validation_needs_no_gpu():
    """hh_lfa_rho / hh_lfa_sigma_c validate before touching the device:
    n = 0 is OK, NULL arrays are HH_E_ARG (1), bad queries or brackets HH_E_CONFIG (2)."""
    lib = _lib()
    out = (ctypes.c_double * 1)()
    assert lib.hh_lfa_rho(None, 0, 0, None) == 0
    assert lib.hh_lfa_rho(None, 1, 0, out) == 1
    bad = [_Q(10.0, 1 / 32, 1.0, 1.0, 0.6, 2, 2, 1, 0),      # m < 2
           _Q(10.0, 0.0, 1.0, 1.0, 0.6, 2, 2, 8, 0),         # h <= 0
           _Q(10.0, 1 / 32, 1.0, 1.0, 1.5, 2, 2, 8, 0),      # omega > 1
           _Q(10.0, 1 / 32, 1.0, 1.0, 0.6, -1, 2, 8, 0)]     # nu < 0
    for q in bad:
        assert lib.hh_lfa_rho(ctypes.byref(q), 1, 0, out) == 2
    ok = _Q(10.0, 1 / 32, 1.0, 1.0, 0.6, 2, 2, 8, 0)
    f = ctypes.c_double
    assert lib.hh_lfa_sigma_c(ctypes.byref(ok), 1, 0, f(2.0), f(1.0), f(1e-2), out) == 2   # lo >= hi
    assert lib.hh_lfa_sigma_c(ctypes.byref(ok), 1, 0, f(1.0), f(2.0), f(0.0), out) == 2    # tol <= 0
    assert lib.hh_lfa_sigma_c(None, 0, 0, f(1.0), f(2.0), f(1e-2), None) == 0
    st = (ctypes.c_double * 4)()
    assert lib.hh_lfa_stats(1, st) == 0 and lib.hh_lfa_stats(0, st) == 0
    assert list(st) == [0.0, 0.0, 0.0, 0.0]
