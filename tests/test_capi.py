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


def test_new_entry_points_validate_without_a_gpu():
    """Argument checks of the WMG coarse-solve and band-path entry points run
    before any CUDA call (no device needed)."""
    from paper_1310_0956_b200 import _native
    lib = _native.load()
    dp = ctypes.c_void_p(8)
    nbytes = ctypes.c_size_t()
    assert lib.wmg_spd_inverse_workspace(2, 256, ctypes.byref(nbytes)) == _native.WMG_OK
    assert nbytes.value == 2 * 2 * (128 * 128 + 2 * 256 * 128) * 8   # two buffer sets
    assert lib.wmg_spd_inverse(1, 100, dp, 100 * 100, dp, dp, None) == _native.WMG_EINVAL
    assert b"multiple of 128" in lib.wmg_last_error()
    assert lib.wmg_spd_inverse(2, 128, dp, 10, dp, dp, None) == _native.WMG_EDIM
    elems = ctypes.c_longlong()
    assert lib.wmg_packed_sym_sizes(3, 384, ctypes.byref(elems), None) == _native.WMG_OK
    assert elems.value == 6 * 128 * 128
    assert lib.wmg_packed_sym_sizes(1, 100, ctypes.byref(elems), None) == _native.WMG_EINVAL
    assert lib.wmg_sym_pack(1, 130, dp, 130 * 130, dp, 1, None) == _native.WMG_EINVAL
    assert lib.wmg_packed_symv(1, 64, dp, 1, dp, 64, dp, 64, dp, None) == _native.WMG_EINVAL
    bands = (ctypes.c_int * 2)(0, 5)
    assert lib.wmg_haar_prolong_path(64, 2, 1, bands, dp, dp, None) == _native.WMG_EINVAL
    assert b"bad band" in lib.wmg_last_error()
    bands = (ctypes.c_int * 2)(0, 3)
    assert lib.wmg_haar_restrict_path(66, 2, 1, bands, dp, dp, None) == _native.WMG_EINVAL
    assert lib.wmg_haar_restrict_path(64, 8, 1, bands, dp, dp, None) == _native.WMG_EINVAL
    assert lib.wmg_haar_prolong_path(64, 2, 0, bands, dp, dp, None) == _native.WMG_OK


def test_fused_cgls_entry_points_validate_without_a_gpu():
    """wmg_det_partials / wmg_cgls_update / wmg_cgls_direction reject what the
    fused kernels cannot do (vectors longer than 2^20, unknown modes, NULL
    buffers) before any CUDA call."""
    from paper_1310_0956_b200 import _native
    lib = _native.load()
    dp = ctypes.c_void_p(8)
    big = (1 << 20) + 1
    upd = lib.wmg_cgls_update
    assert upd(100, big, dp, dp, dp, dp, dp, None, 0.0, dp, None) == _native.WMG_EINVAL
    assert b"2^20" in lib.wmg_last_error()
    assert upd(big, 100, dp, dp, dp, dp, dp, None, 0.0, dp, None) == _native.WMG_EINVAL
    assert upd(0, 100, dp, dp, dp, dp, dp, None, 0.0, dp, None) == _native.WMG_EINVAL
    assert upd(100, 100, None, dp, dp, dp, dp, None, 0.0, dp, None) == _native.WMG_EINVAL
    assert upd(100, 100, dp, dp, dp, dp, dp, None, 0.5, dp, None) == _native.WMG_EINVAL
    assert b"<p,p>" in lib.wmg_last_error()
    assert lib.wmg_cgls_direction(big, dp, dp, dp, 1, dp, None) == _native.WMG_EINVAL
    assert lib.wmg_cgls_direction(100, dp, dp, dp, 3, dp, None) == _native.WMG_EINVAL
    assert b"mode" in lib.wmg_last_error()
    assert lib.wmg_cgls_direction(100, dp, dp, None, 1, dp, None) == _native.WMG_EINVAL
    ops = (ctypes.c_int * 1)(4)
    a = (ctypes.c_void_p * 1)(8)
    assert lib.wmg_det_partials(0, 1, ops, a, None, None, dp, None) == _native.WMG_EINVAL
    assert lib.wmg_det_partials(100, 0, ops, a, None, None, dp, None) == _native.WMG_EINVAL
    bad = (ctypes.c_int * 1)(7)
    assert lib.wmg_det_partials(100, 1, bad, a, None, None, dp, None) == _native.WMG_EINVAL
    dot = (ctypes.c_int * 1)(0)                        # RED_DOT needs a second operand
    assert lib.wmg_det_partials(100, 1, dot, a, None, None, dp, None) == _native.WMG_EINVAL
