"""The C-ABI library loads and exports every symbol include/wmgb200.h declares
(no compute calls -- this runs without a GPU)."""
import ctypes
import os
import re

from conftest import ROOT


def header_symbols():
    with open(os.path.join(ROOT, "include", "wmgb200.h")) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"\b(wmg_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_expected_entry_points():
    syms = header_symbols()
    for s in ("wmg_geometry_create", "wmg_forward", "wmg_backward", "wmg_row_sums",
              "wmg_col_sums", "wmg_det_reduce", "wmg_haar_restrict", "wmg_haar_prolong",
              "wmg_leaf_factor"):
        assert s in syms


def test_library_exports_every_header_symbol():
    from paper_1310_0956_b200 import _native
    if not os.path.exists(_native.LIB_PATH):
        _native.build()
    lib = ctypes.CDLL(_native.LIB_PATH)
    missing = [s for s in header_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    # the Python binding declares a signature for every exported symbol
    assert set(header_symbols()) == set(_native.EXPORTED)
    assert lib.wmg_version() == 1


def test_invalid_arguments_map_to_errors():
    from paper_1310_0956_b200 import _native
    lib = _native.load()
    h = ctypes.c_void_p()
    c = (ctypes.c_double * 1)(1.0)
    s = (ctypes.c_double * 1)(0.0)
    rc = lib.wmg_geometry_create(0, 4, 1, c, s, ctypes.byref(h))
    assert rc == _native.WMG_EINVAL
    assert b"positive" in lib.wmg_last_error()
    rc = lib.wmg_haar_restrict(3, ctypes.c_void_p(8), 1, ctypes.c_void_p(8), None)
    assert rc == _native.WMG_EINVAL
