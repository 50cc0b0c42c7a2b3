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
