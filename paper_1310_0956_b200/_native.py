"""ctypes binding of ``lib/libwmgb200.so`` (the C ABI in ``include/wmgb200.h``).

There is deliberately no fallback: if the CUDA library or a GPU is missing the
product path raises ``RuntimeError`` instead of computing anything on the CPU.
Error codes map onto the exception classes the reference raises
(/root/reference/pkg/src/wmgtomo/sparse_kernels.py:22-27).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

from .sparse_kernels import DimensionMismatchError, NotPositiveDefiniteError

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "lib", "libwmgb200.so")
CSRC = os.path.join(_PKG, "csrc")

WMG_OK, WMG_EINVAL, WMG_EDIM, WMG_ENOTSPD, WMG_ECUDA = range(5)
MODE_PARITY, MODE_FAST = 0, 1
F32, F64 = 0, 1
KERNEL_LINE, KERNEL_JOSEPH = 0, 1
RED_DOT, RED_SQDIFF, RED_SUM, RED_DOTDIFF, RED_SQ = range(5)

_lib = None

_vp = ctypes.c_void_p
_dp = ctypes.c_void_p      # device pointers are passed as plain integers
_i = ctypes.c_int
_ll = ctypes.c_longlong
_d = ctypes.c_double

_SIGS = {
    "wmg_version": (_i, []),
    "wmg_last_error": (ctypes.c_char_p, []),
    "wmg_geometry_create": (_i, [_i, _i, _i, ctypes.POINTER(_d), ctypes.POINTER(_d),
                                 ctypes.POINTER(_vp)]),
    "wmg_geometry_destroy": (_i, [_vp]),
    "wmg_geometry_shape": (_i, [_vp, ctypes.POINTER(_ll), ctypes.POINTER(_ll)]),
    "wmg_geometry_symmetry": (_i, [_vp, _i, ctypes.POINTER(_i)]),
    "wmg_geometry_transposition": (_i, [_vp, ctypes.POINTER(_i)]),
    "wmg_geometry_kernel": (_i, [_vp, _i, ctypes.POINTER(_i)]),
    "wmg_forward_workspace": (_i, [_vp, _i, _i, ctypes.POINTER(ctypes.c_size_t)]),
    "wmg_forward": (_i, [_vp, _i, _i, _i, _i, _dp, _dp, _dp, _dp, _vp]),
    "wmg_backward": (_i, [_vp, _i, _i, _i, _i, _dp, _dp, _i, _dp, _vp]),
    "wmg_backward_bands": (_i, [_vp, _i, ctypes.POINTER(_i)]),
    "wmg_backward_band": (_i, [_vp, _i, _i, _i, _dp, _dp, _i, _i, _vp]),
    "wmg_forward_batch": (_i, [_vp, _i, _i, _i, _i, _dp, _dp, _i, _dp, _vp]),
    "wmg_backward_batch": (_i, [_vp, _i, _i, _i, _i, _dp, _dp, _i, _i, _vp]),
    "wmg_row_sums": (_i, [_vp, _dp, _vp]),
    "wmg_col_sums": (_i, [_vp, _dp, _vp]),
    "wmg_csr_counts": (_i, [_vp, _dp, _dp, _vp]),
    "wmg_csr_fill": (_i, [_vp, _dp, _dp, _dp, _vp]),
    "wmg_det_scratch_len": (_ll, [_ll, _i]),
    "wmg_det_reduce": (_i, [_ll, _i, ctypes.POINTER(_i), ctypes.POINTER(_vp),
                            ctypes.POINTER(_vp), ctypes.POINTER(_vp), _dp, _dp, _vp]),
    "wmg_maxabs": (_i, [_ll, _dp, _dp, _dp, _vp]),
    "wmg_axpy": (_i, [_ll, _dp, _dp, _d, _i, _dp, _vp]),
    "wmg_lincomb": (_i, [_ll, _dp, _d, _dp, _d, _dp, _d, _dp, _vp]),
    "wmg_bicg_p": (_i, [_ll, _dp, _dp, _d, _d, _dp, _vp]),
    "wmg_bicg_x": (_i, [_ll, _dp, _d, _dp, _d, _dp, _vp]),
    "wmg_scale": (_i, [_ll, _dp, _d, _dp, _dp, _vp]),
    "wmg_recip": (_i, [_ll, _dp, _dp, _vp]),
    "wmg_smooth_update": (_i, [_ll, _dp, _d, _dp, _dp, _dp, _vp]),
    "wmg_sirt_update": (_i, [_ll, _dp, _dp, _dp, _d, _vp]),
    "wmg_add_scaled": (_i, [_ll, _dp, _dp, _d, _i, _dp, _vp]),
    "wmg_cgs_update": (_i, [_ll, _i, _dp, _dp, _ll, _dp, _vp]),
    "wmg_combo": (_i, [_ll, _i, _dp, _dp, _ll, _dp, _i, _vp]),
    "wmg_cast": (_i, [_ll, _i, _dp, _dp, _vp]),
    "wmg_h2d_staged": (_i, [_vp, _vp, ctypes.c_size_t, _vp, _i, _vp]),
    "wmg_axpy_dev": (_i, [_ll, _dp, _dp, _dp, _i, _dp, _vp]),
    "wmg_lincomb_dev": (_i, [_ll, _dp, _d, _dp, _dp, _dp, _vp]),
    "wmg_cgls_scalars": (_i, [_dp, _d, _i, _vp]),
    "wmg_det_partials": (_i, [_ll, _i, ctypes.POINTER(_i), ctypes.POINTER(_vp),
                              ctypes.POINTER(_vp), ctypes.POINTER(_vp), _dp, _vp]),
    "wmg_cgls_update": (_i, [_ll, _ll, _dp, _dp, _dp, _dp, _dp, _dp, _d, _dp, _vp]),
    "wmg_cgls_direction": (_i, [_ll, _dp, _dp, _dp, _i, _dp, _vp]),
    "wmg_batched_gemv": (_i, [_i, _i, _dp, _ll, _dp, _ll, _dp, _ll, _vp]),
    "wmg_haar_restrict": (_i, [_i, _dp, _i, _dp, _vp]),
    "wmg_haar_prolong": (_i, [_i, _dp, _i, _dp, _i, _vp]),
    "wmg_haar_restrict_batch": (_i, [_i, _i, _dp, _i, _dp, _vp]),
    "wmg_forward_path_supported": (_i, [_vp, _i, ctypes.POINTER(_i)]),
    "wmg_forward_path": (_i, [_vp, _dp, _i, _i, ctypes.POINTER(_i), _dp, _dp, _vp]),
    "wmg_haar_prolong_batch": (_i, [_i, _i, _i, ctypes.POINTER(_i), _dp, _dp, _i, _vp]),
    "wmg_smooth_update_batch": (_i, [_ll, _i, _dp, ctypes.POINTER(_d), ctypes.POINTER(_vp), _dp,
                                     _dp, _vp]),
    "wmg_haar_prolong_path": (_i, [_i, _i, _i, ctypes.POINTER(_i), _dp, _dp, _vp]),
    "wmg_haar_restrict_path": (_i, [_i, _i, _i, ctypes.POINTER(_i), _dp, _dp, _vp]),
    "wmg_leaf_factor": (_i, [_vp, _i, ctypes.POINTER(_i), _ll, _ll, _dp, _vp]),
    "wmg_leaf_gram": (_i, [_vp, _i, ctypes.POINTER(_i), _dp, _dp, _vp]),
    "wmg_spd_inverse_workspace": (_i, [_i, _i, ctypes.POINTER(ctypes.c_size_t)]),
    "wmg_spd_inverse": (_i, [_i, _i, _dp, _ll, _dp, _dp, _vp]),
    "wmg_cholesky_dinv_elems": (_i, [_i, ctypes.POINTER(_ll)]),
    "wmg_cholesky_factor": (_i, [_i, _i, _dp, _ll, _dp, _dp, _vp]),
    "wmg_cholesky_solve": (_i, [_i, _i, _dp, _ll, _dp, _dp, _ll, _i, _vp]),
    "wmg_packed_sym_sizes": (_i, [_i, _i, ctypes.POINTER(_ll), ctypes.POINTER(ctypes.c_size_t)]),
    "wmg_sym_pack": (_i, [_i, _i, _dp, _ll, _dp, _ll, _vp]),
    "wmg_packed_symv": (_i, [_i, _i, _dp, _ll, _dp, _ll, _dp, _ll, _dp, _vp]),
}

EXPORTED = tuple(_SIGS)


def build(quiet: bool = True) -> str:
    """Compile the CUDA library for sm_100a (nvcc cross-compiles without a GPU)."""
    cmd = ["make", "-C", CSRC, "-j8"]
    if quiet:
        cmd.insert(1, "-s")
    subprocess.run(cmd, check=True)
    return LIB_PATH


def load(require_gpu: bool = False):
    """Load the library (no GPU needed just to load and inspect symbols)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"libwmgb200.so not built ({LIB_PATH}); run __graft_entry__.build() -- "
                "there is no CPU fallback for the B200 hot path")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    if require_gpu:
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("no CUDA device: the B200 hot path has no CPU fallback")
    return _lib


def check(rc: int, what: str = ""):
    if rc == WMG_OK:
        return
    msg = (_lib.wmg_last_error() or b"").decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == WMG_EDIM:
        raise DimensionMismatchError(text)
    if rc == WMG_ENOTSPD:
        raise NotPositiveDefiniteError(text)
    if rc == WMG_EINVAL:
        raise ValueError(text)
    raise RuntimeError(text)


def call(name: str, *args):
    L = load()
    check(getattr(L, name)(*args), name)
