"""ctypes front end of the C oracle (``oracle/wmg_oracle.c``) -- test-only.

Restates /root/reference/pkg/src/wmgtomo/geometry.py:88-215 (``_line_entries``,
``build_projector``, ``apply``, ``apply_transpose``) and the scalings of
solvers.py:79-86.  Built by ``oracle/Makefile`` into ``oracle/_build``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np
import scipy.sparse as sp

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None

_dp = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)


def build():
    """Compile the oracle (gcc, no FMA contraction)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.orc_row_counts.restype = ctypes.c_int64
        L.orc_row_counts.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp, _dp, _i64p]
        L.orc_fill_csr.restype = ctypes.c_int
        L.orc_fill_csr.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp, _dp, _i64p,
                                   _i64p, _dp]
        L.orc_forward.restype = ctypes.c_int
        L.orc_forward.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp, _dp, _dp, _dp]
        L.orc_backward.restype = ctypes.c_int
        L.orc_backward.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp, _dp, _dp, _dp]
        L.orc_csr_matvec.restype = ctypes.c_int
        L.orc_csr_matvec.argtypes = [ctypes.c_int64, _i64p, _i64p, _dp, _dp, _dp]
        L.orc_csr_row_sums.restype = None
        L.orc_csr_row_sums.argtypes = [ctypes.c_int64, _i64p, _dp, _dp]
        L.orc_reduceat_segment.restype = ctypes.c_double
        L.orc_reduceat_segment.argtypes = [_dp, ctypes.c_int64]
        L.orc_set_threads.restype = ctypes.c_int
        L.orc_set_threads.argtypes = [ctypes.c_int]
        L.orc_set_kernel.restype = ctypes.c_int
        L.orc_set_kernel.argtypes = [ctypes.c_int]
        L.orc_num_threads.restype = ctypes.c_int
        L.orc_num_threads.argtypes = []
        _lib = L
    return _lib


def _p(a, t=_dp):
    return a.ctypes.data_as(t)


def snapped_trig(angles):
    """geometry.py:77-85 vectorised: residues below 1e-15 snap to exact 0/+-1."""
    a = np.asarray(angles, dtype=np.float64)
    c = np.array([float(np.cos(t)) for t in a])
    s = np.array([float(np.sin(t)) for t in a])
    for i in range(a.size):
        if abs(c[i]) < 1e-15:
            c[i], s[i] = 0.0, float(np.sign(s[i]))
        elif abs(s[i]) < 1e-15:
            c[i], s[i] = float(np.sign(c[i])), 0.0
    return c, s


def equiangular(n_angles):
    """geometry.py:72: angles = arange(m) * (pi / m)."""
    return np.arange(n_angles) * (np.pi / n_angles)


def set_threads(t: int):
    lib().orc_set_threads(int(t))


def num_threads() -> int:
    return int(lib().orc_num_threads())


KERNELS = {"line": 0, "joseph": 1}


def build_csr(n, d, angles, return_dups=False, kernel="line"):
    """The reference W (CSR, float64, int64 indices) for an arbitrary angle list
    (``kernel``: "line" = geometry.py:88-128, "joseph" = geometry.py:131-175)."""
    lib().orc_set_kernel(KERNELS[kernel])
    try:
        return _build_csr(n, d, angles, return_dups)
    finally:
        lib().orc_set_kernel(0)


def _build_csr(n, d, angles, return_dups):
    c, s = snapped_trig(angles)
    m = c.size
    counts = np.zeros(m * d, dtype=np.int64)
    dups = lib().orc_row_counts(n, d, m, _p(c), _p(s), _p(counts, _i64p))
    if dups < 0:
        raise MemoryError("oracle scratch allocation failed")
    indptr = np.zeros(m * d + 1, dtype=np.int64)
    np.cumsum(counts, out=indptr[1:])
    nnz = int(indptr[-1])
    indices = np.empty(nnz, dtype=np.int64)
    data = np.empty(nnz, dtype=np.float64)
    if lib().orc_fill_csr(n, d, m, _p(c), _p(s), _p(indptr, _i64p), _p(indices, _i64p),
                          _p(data)) != 0:
        raise MemoryError("oracle scratch allocation failed")
    w = sp.csr_matrix((data, indices, indptr), shape=(m * d, n * n))
    return (w, int(dups)) if return_dups else w


def forward(n, d, angles, x):
    c, s = snapped_trig(angles)
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty(c.size * d)
    lib().orc_forward(n, d, c.size, _p(c), _p(s), _p(x), _p(y))
    return y


def backward(n, d, angles, y):
    c, s = snapped_trig(angles)
    y = np.ascontiguousarray(y, dtype=np.float64)
    x = np.empty(n * n)
    lib().orc_backward(n, d, c.size, _p(c), _p(s), _p(y), _p(x))
    return x


def csr_matvec(a: sp.csr_matrix, x):
    """csr_matvec order (bitwise scipy) with all host threads."""
    indptr = np.ascontiguousarray(a.indptr, dtype=np.int64)
    indices = np.ascontiguousarray(a.indices, dtype=np.int64)
    data = np.ascontiguousarray(a.data, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty(a.shape[0])
    lib().orc_csr_matvec(a.shape[0], _p(indptr, _i64p), _p(indices, _i64p), _p(data), _p(x),
                         _p(y))
    return y


def row_sums(w: sp.csr_matrix):
    """np.add.reduceat semantics (solvers.py:81 via scipy _minor_reduce)."""
    indptr = np.ascontiguousarray(w.indptr, dtype=np.int64)
    data = np.ascontiguousarray(w.data, dtype=np.float64)
    out = np.empty(w.shape[0])
    lib().orc_csr_row_sums(w.shape[0], _p(indptr, _i64p), _p(data), _p(out))
    return out


def col_sums(w: sp.csr_matrix):
    """ones @ W == W^T 1 summed in ascending ray order (solvers.py:82)."""
    return w.T @ np.ones(w.shape[0])
