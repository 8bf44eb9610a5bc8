"""Parallel-beam geometry and the matrix-free line-intersection projector on B200.

Drop-in for /root/reference/pkg/src/wmgtomo/geometry.py:
  * ``Geometry`` / ``build_geometry`` (:34-74) -- identical validation and
    angle grid ``arange(m) * (pi / m)``;
  * ``build_projector(g, kernel="line")`` (:178-197) returns a ``LineProjector``
    instead of a scipy CSR.  It implements the subset of the scipy protocol the
    reference solvers use: ``shape``, ``@``, ``.T``,
    ``.tocsr()``, ``.sum(axis)``; W is never materialised -- the weights are
    recomputed by the sm_100a kernels on every application;
  * ``apply`` / ``apply_transpose`` (:200-215) with the same
    ``DimensionMismatchError`` contract.

Numerics.  ``precision="float64"`` (default) runs the PARITY kernels: weights,
pixel assignment and summation orders are bit-identical to the reference CSR and
scipy's csr_matvec / csc_matvec.  ``precision="float32"`` runs the FAST kernels
(fp32 data and accumulation, 64-bit fixed-point geometry), within 1e-5 relative
of the float64 reference.  ``mode="fast"`` with float64 selects the fast kernels
in float64 arithmetic.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _device as D
from . import _native as N
from .sparse_kernels import DimensionMismatchError


@dataclass(frozen=True)
class Geometry:
    """Parallel-beam scan description: n-by-n grid, m angles, rays per angle."""

    n_pixels_per_side: int
    n_detectors: int
    n_angles: int
    angles: np.ndarray = field(repr=False)
    pixel_size: float = 1.0
    detector_spacing: float = 1.0

    def __post_init__(self):
        if self.n_pixels_per_side < 1 or self.n_detectors < 1 or self.n_angles < 1:
            raise ValueError("geometry dimensions must be positive")
        a = np.asarray(self.angles, dtype=np.float64)
        if a.shape != (self.n_angles,):
            raise ValueError("angles length must equal n_angles")
        if np.any(a < 0.0) or np.any(a >= np.pi):
            raise ValueError("angles must lie in [0, pi)")
        if np.any(np.diff(a) <= 0.0):
            raise ValueError("angles must be strictly increasing")
        if self.pixel_size != 1.0 or self.detector_spacing != 1.0:
            # the reference hard-wires unit pixels (geometry.py:92-95)
            raise ValueError("only unit pixel size and detector spacing are supported")
        object.__setattr__(self, "angles", a)

    @property
    def n_image(self) -> int:
        return self.n_pixels_per_side ** 2

    @property
    def n_data(self) -> int:
        return self.n_angles * self.n_detectors

    def subset(self, index) -> "Geometry":
        """Geometry restricted to a subset of the angles (rows of W)."""
        a = self.angles[np.asarray(index)]
        return Geometry(self.n_pixels_per_side, self.n_detectors, a.size, angles=a)


def build_geometry(n: int, n_detectors: int, n_angles: int) -> Geometry:
    """Equiangular geometry over the half-turn [0, pi) (geometry.py:68-74)."""
    if n < 1 or n_detectors < 1 or n_angles < 1:
        raise ValueError("all geometry arguments must be >= 1")
    angles = np.arange(n_angles) * (np.pi / n_angles)
    return Geometry(n_pixels_per_side=n, n_detectors=n_detectors,
                    n_angles=n_angles, angles=angles)


def snapped_trig(angles):
    """geometry.py:77-85, evaluated on the host with numpy for every angle."""
    a = np.asarray(angles, dtype=np.float64)
    c = np.cos(a)
    s = np.sin(a)
    for i in range(a.size):
        ci, si = float(np.cos(a[i])), float(np.sin(a[i]))
        if abs(ci) < 1e-15:
            ci, si = 0.0, float(np.sign(si))
        elif abs(si) < 1e-15:
            ci, si = float(np.sign(ci)), 0.0
        c[i], s[i] = ci, si
    return np.ascontiguousarray(c), np.ascontiguousarray(s)


_PRECISIONS = {"float64": N.F64, "fp64": N.F64, "double": N.F64,
               "float32": N.F32, "fp32": N.F32, "float": N.F32}


_PENDING_DESTROY = []


def _destroy_geometry(h):
    """Free a device geometry, unless a CUDA graph capture is running on this
    thread (the garbage collector may finalise a projector mid-capture, and a
    cudaFree would invalidate the capture): then defer to the next call."""
    t = D.torch()
    try:
        capturing = t.cuda.is_current_stream_capturing()
    except Exception:  # pragma: no cover
        capturing = False
    if capturing:
        _PENDING_DESTROY.append(h)
        return
    lib = N.load()
    while _PENDING_DESTROY:
        lib.wmg_geometry_destroy(_PENDING_DESTROY.pop())
    if h is not None:
        lib.wmg_geometry_destroy(h)


class LineProjector:
    """Matrix-free W (M x N) with the reference line-intersection weights."""

    format = "matrix-free"

    def __init__(self, g: Geometry, precision: str = "float64", mode: str | None = None,
                 device=None, kernel: str = "line"):
        t = D.require_cuda()
        self.kernel = kernel
        if precision not in _PRECISIONS:
            raise ValueError(f"unknown precision '{precision}'")
        self.geometry = g
        self.precision = _PRECISIONS[precision]
        if mode is None:
            mode = "parity" if self.precision == N.F64 else "fast"
        if mode not in ("parity", "fast"):
            raise ValueError(f"unknown mode '{mode}'")
        if mode == "parity" and self.precision != N.F64:
            raise ValueError("parity mode is float64 only")
        self.mode = mode
        self._mode_code = N.MODE_PARITY if mode == "parity" else N.MODE_FAST
        self.device = t.device(device) if device is not None else t.device("cuda",
                                                                        t.cuda.current_device())
        self.n = g.n_pixels_per_side
        self.shape = (g.n_data, g.n_image)
        self.dtype = np.float64
        c, s = snapped_trig(g.angles)
        self._cos, self._sin = c, s
        handle = N.ctypes.c_void_p()
        if _PENDING_DESTROY:
            _destroy_geometry(None)
        with t.cuda.device(self.device):
            N.call("wmg_geometry_create", self.n, g.n_detectors, g.n_angles,
                   c.ctypes.data_as(N.ctypes.POINTER(N.ctypes.c_double)),
                   s.ctypes.data_as(N.ctypes.POINTER(N.ctypes.c_double)),
                   N.ctypes.byref(handle))
        self._h = handle
        if kernel == "joseph":
            N.call("wmg_geometry_kernel", handle, N.KERNEL_JOSEPH, None)
        self._ws = {}
        self._anomaly = t.zeros(1, dtype=t.int32, device=self.device)
        self._sums = {}

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _destroy_geometry(h)
            except Exception:  # pragma: no cover - interpreter shutdown
                pass
            self._h = None

    # ---------------------------------------------------------------- helpers
    @property
    def handle(self):
        return self._h

    @property
    def T(self):
        return _Transposed(self)

    @property
    def symmetric(self) -> bool:
        """Whether the fast kernels share weights across mirror images."""
        st = N.ctypes.c_int()
        N.call("wmg_geometry_symmetry", self._h, -1, N.ctypes.byref(st))
        return bool(st.value)

    @property
    def transposition_closed(self) -> bool:
        """Whether the angle set is also closed under theta -> pi/2 - theta (the
        backprojector then shares each weight among eight pixel/angle pairs)."""
        st = N.ctypes.c_int()
        N.call("wmg_geometry_transposition", self._h, N.ctypes.byref(st))
        return bool(st.value)

    def set_symmetry(self, enable) -> bool:
        """Enable (True: where profitable), force ("force": at every size; "tma":
        forced with the experimental TMA-staged forward) or disable (False) the
        mirror-symmetry kernels; no-op if the angle set is not symmetric.
        Returns whether it is enabled."""
        code = {"force": 2, "tma": 4, "rowlayout": 10, "fwd1": 18, "lockstep": 34, "fwdrows": 66, "plainplanes": 130, "bwd8x4": 258, "bwdrun32": 514, "bwdrun64": 1026, "bwdsym8": 8194, "bwdrun": 16386, "bwdrunflat": 49154, "fwdflat": 65538}.get(enable, None)
        if code is None:
            code = int(bool(enable))
        st = N.ctypes.c_int()
        N.call("wmg_geometry_symmetry", self._h, code, N.ctypes.byref(st))
        self._ws.pop("path_ok", None)         # the fused path forward follows the dispatch
        return bool(st.value)

    def prefer_concurrent(self, on: bool = True) -> bool:
        """Throughput dispatch for callers that run several products concurrently
        on different streams (slice stacks): keeps the forward in its unsplit
        four-octet blocks.  Launches of few blocks (n >= 1792 with few angles)
        otherwise take the 8-segment form, which is faster alone (its blocks drain
        evenly) but slower when another stream's kernels fill the tails anyway
        (config-4 geometry: 2.15 vs 2.23 ms per pair alone, 1.94 vs 1.88 ms per
        pair with two streams, tools/probe_cfg4_pair.py)."""
        return self.set_symmetry("fwdflat" if on else True)

    def tocsr(self):
        return self

    def _workspace(self, tin_code):
        t = D.torch()
        ws = self._ws.get(tin_code)
        if ws is None:
            nbytes = N.ctypes.c_size_t()
            N.call("wmg_forward_workspace", self._h, self.precision, tin_code,
                   N.ctypes.byref(nbytes))
            # zero-initialised once: the padded margins are never written again
            ws = t.zeros((nbytes.value + 7) // 8, dtype=t.float64, device=self.device)
            self._ws[tin_code] = ws
        return ws

    @staticmethod
    def _code(tensor):
        t = D.torch()
        if tensor.dtype == t.float64:
            return N.F64
        if tensor.dtype == t.float32:
            return N.F32
        raise TypeError(f"unsupported dtype {tensor.dtype}")

    def _io_dtype(self, v):
        """Vector dtype of a call: float64 (the reference's convention), except
        that a float32 projector keeps float32 vectors float32 (CUDA tensors or
        numpy arrays) -- half the bytes over PCIe and in HBM."""
        t = D.torch()
        if self.precision == N.F32:
            if D.is_torch(v) and v.dtype == t.float32:
                return t.float32
            if isinstance(v, np.ndarray) and v.dtype == np.float32:
                return t.float32
        return t.float64 if (self.precision == N.F64 or not D.is_torch(v)) else v.dtype

    # ------------------------------------------------------------ operators
    def forward_(self, x, out, anomaly=None):
        """out = W x on device tensors (float32/float64 as the mode allows)."""
        tin, tout = self._code(x), self._code(out)
        if x.numel() != self.shape[1]:
            raise DimensionMismatchError(
                f"apply: vector length {x.numel()} != n_cols {self.shape[1]}")
        if out.numel() != self.shape[0]:
            raise DimensionMismatchError("apply: output length mismatch")
        ws = self._workspace(tin) if self._mode_code == N.MODE_FAST else None
        N.call("wmg_forward", self._h, self._mode_code, self.precision, tin, tout,
               D.ptr(x), D.ptr(out), D.ptr(ws), D.ptr(anomaly), D.stream_handle())
        return out

    def forward_batch_(self, X, OUT):
        """OUT[b] = W X[b] for a contiguous batch (B, n*n) -> (B, M) on the device."""
        t = D.torch()
        B = X.shape[0]
        if X.numel() != B * self.shape[1] or OUT.numel() != B * self.shape[0]:
            raise DimensionMismatchError("forward_batch_: shape mismatch")
        tin, tout = self._code(X), self._code(OUT)
        ws = None
        if self._mode_code == N.MODE_FAST:
            key = ("batch", tin, B)
            ws = self._ws.get(key)
            if ws is None:
                nbytes = N.ctypes.c_size_t()
                N.call("wmg_forward_workspace", self._h, self.precision, tin,
                       N.ctypes.byref(nbytes))
                ws = t.zeros((B * nbytes.value + 7) // 8, dtype=t.float64, device=self.device)
                self._ws[key] = ws
        N.call("wmg_forward_batch", self._h, self._mode_code, self.precision, tin, tout,
               D.ptr(X), D.ptr(OUT), B, D.ptr(ws), D.stream_handle())
        return OUT

    @property
    def supports_forward_path(self) -> bool:
        """Whether forward_path_ (prolongation fused into the forward) is available."""
        v = self._ws.get("path_ok")
        if v is None:
            ok = N.ctypes.c_int()
            N.call("wmg_forward_path_supported", self._h, self.precision, N.ctypes.byref(ok))
            v = self._ws["path_ok"] = bool(ok.value) and self._mode_code == N.MODE_FAST
        return v

    def forward_path_(self, C, paths, OUT):
        """OUT[b] = W R_{paths[b]}^T C[b] (float64 fast mode, small grids): the
        WMG node prolongation (multilevel.py:109-113) evaluated inside the forward's
        padding pass, bit-identical to prolong_path + forward_batch_."""
        t = D.torch()
        B = C.shape[0]
        depth = len(paths[0])
        ws = self._ws.get(("batch", N.F64, B))
        if ws is None:
            nbytes = N.ctypes.c_size_t()
            N.call("wmg_forward_workspace", self._h, self.precision, N.F64, N.ctypes.byref(nbytes))
            ws = t.zeros((B * nbytes.value + 7) // 8, dtype=t.float64, device=self.device)
            self._ws[("batch", N.F64, B)] = ws
        from .multilevel import BAND_CODE
        codes = (N.ctypes.c_int * (B * depth))(*[BAND_CODE[b] for p in paths for b in p])
        N.call("wmg_forward_path", self._h, D.ptr(C), depth, B, codes, D.ptr(OUT), D.ptr(ws),
               D.stream_handle())
        return OUT

    def backward_batch_(self, Y, OUT, accumulate=False):
        """OUT[b] (+)= W^T Y[b] for a contiguous batch (B, M) -> (B, n*n)."""
        B = Y.shape[0]
        if Y.numel() != B * self.shape[0] or OUT.numel() != B * self.shape[1]:
            raise DimensionMismatchError("backward_batch_: shape mismatch")
        N.call("wmg_backward_batch", self._h, self._mode_code, self.precision, self._code(Y),
               self._code(OUT), D.ptr(Y), D.ptr(OUT), B, int(bool(accumulate)),
               D.stream_handle())
        return OUT

    def backward_(self, y, out, accumulate=False, anomaly=None):
        """out (+)= W^T y on device tensors."""
        tin, tout = self._code(y), self._code(out)
        if y.numel() != self.shape[0]:
            raise DimensionMismatchError(
                f"apply_transpose: vector length {y.numel()} != n_rows {self.shape[0]}")
        if out.numel() != self.shape[1]:
            raise DimensionMismatchError("apply_transpose: output length mismatch")
        N.call("wmg_backward", self._h, self._mode_code, self.precision, tin, tout, D.ptr(y),
               D.ptr(out), int(bool(accumulate)), D.ptr(anomaly), D.stream_handle())
        return out

    def backward_bands(self) -> int:
        """Number of row bands of the banded backprojection (0: not available
        for this geometry / precision; see wmg_backward_band)."""
        nb = N.ctypes.c_int()
        N.call("wmg_backward_bands", self._h, self.precision, N.ctypes.byref(nb))
        return nb.value if self._mode_code == N.MODE_FAST else 0

    def backward_band_(self, y, out, band0: int, band1: int):
        """Bands [band0, band1) of out = W^T y: image rows [32 band0, 32 band1)
        and [n - 32 band1, n - 32 band0) complete (bit-identical to backward_).
        Bands must be issued in increasing order on one stream."""
        if y.numel() != self.shape[0] or out.numel() != self.shape[1]:
            raise DimensionMismatchError("backward_band_: length mismatch")
        N.call("wmg_backward_band", self._h, self.precision, self._code(y), self._code(out),
               D.ptr(y), D.ptr(out), int(band0), int(band1), D.stream_handle())
        return out

    def forward(self, x):
        t = D.torch()
        dt = self._io_dtype(x)
        xd, was_np = D.to_device(x, dt, self.device)
        if xd.dim() != 1:
            xd = xd.reshape(-1)
        if xd.numel() != self.shape[1]:
            raise DimensionMismatchError(
                f"apply: vector length {xd.numel()} != n_cols {self.shape[1]}")
        out = t.empty(self.shape[0], dtype=dt, device=self.device)
        self.forward_(xd, out)
        return D.to_caller(out, was_np)

    def backward(self, y):
        t = D.torch()
        dt = self._io_dtype(y)
        yd, was_np = D.to_device(y, dt, self.device)
        if yd.dim() != 1:
            yd = yd.reshape(-1)
        if yd.numel() != self.shape[0]:
            raise DimensionMismatchError(
                f"apply_transpose: vector length {yd.numel()} != n_rows {self.shape[0]}")
        out = t.empty(self.shape[1], dtype=dt, device=self.device)
        self.backward_(yd, out)
        return D.to_caller(out, was_np)

    def __matmul__(self, v):
        return self.forward(v)

    def dot(self, v):
        return self.forward(v)

    # ------------------------------------------------------------ scalings
    def row_sums_dev(self):
        """Row sums with the reference's np.add.reduceat semantics (device)."""
        t = D.torch()
        r = self._sums.get("rows")
        if r is None:
            r = t.empty(self.shape[0], dtype=t.float64, device=self.device)
            N.call("wmg_row_sums", self._h, D.ptr(r), D.stream_handle())
            self._sums["rows"] = r
        return r

    def col_sums_dev(self):
        """Column sums = ones @ W (device)."""
        t = D.torch()
        c = self._sums.get("cols")
        if c is None:
            c = t.empty(self.shape[1], dtype=t.float64, device=self.device)
            N.call("wmg_col_sums", self._h, D.ptr(c), D.stream_handle())
            self._sums["cols"] = c
        return c

    def sum(self, axis=None):
        if axis in (1, -1):
            return self.row_sums_dev().cpu().numpy()
        if axis in (0, -2):
            return self.col_sums_dev().cpu().numpy()
        if axis is None:
            return float(self.row_sums_dev().sum().item())
        raise ValueError(f"bad axis {axis}")

    # ------------------------------------------------------------ exports
    def csr_device(self):
        """Exact CSR of W assembled on the GPU: (indptr, indices, data) tensors."""
        t = D.torch()
        M = self.shape[0]
        counts = t.empty(M, dtype=t.int64, device=self.device)
        anomaly = t.zeros(1, dtype=t.int32, device=self.device)
        N.call("wmg_csr_counts", self._h, D.ptr(counts), D.ptr(anomaly), D.stream_handle())
        indptr = t.zeros(M + 1, dtype=t.int64, device=self.device)
        t.cumsum(counts, 0, out=indptr[1:])
        nnz = int(indptr[-1].item())
        cols = t.empty(max(nnz, 1), dtype=t.int64, device=self.device)
        vals = t.empty(max(nnz, 1), dtype=t.float64, device=self.device)
        N.call("wmg_csr_fill", self._h, D.ptr(indptr), D.ptr(cols), D.ptr(vals),
               D.stream_handle())
        return indptr, cols[:nnz], vals[:nnz], int(anomaly.item())

    def to_scipy(self):
        """Exact scipy CSR (small n only; for oracle comparisons)."""
        import scipy.sparse as sp
        indptr, cols, vals, _ = self.csr_device()
        return sp.csr_matrix((vals.cpu().numpy(), cols.cpu().numpy(), indptr.cpu().numpy()),
                             shape=self.shape)

    def nnz(self) -> int:
        """Exact number of stored entries of W (the reference CSR's nnz), from a
        GPU counting pass of the exact walker (no CSR is formed)."""
        t = D.torch()
        counts = t.empty(self.shape[0], dtype=t.int64, device=self.device)
        anomaly = t.zeros(1, dtype=t.int32, device=self.device)
        N.call("wmg_csr_counts", self._h, D.ptr(counts), D.ptr(anomaly), D.stream_handle())
        return int(counts.sum().item())

    def anomaly_count(self):
        """Parity-walk consistency counter over one forward + backward pass."""
        t = D.torch()
        a = t.zeros(1, dtype=t.int32, device=self.device)
        x = t.zeros(self.shape[1], dtype=t.float64, device=self.device)
        y = t.zeros(self.shape[0], dtype=t.float64, device=self.device)
        if self.mode == "parity":
            self.forward_(x, y, anomaly=a)
            self.backward_(y, x, anomaly=a)
        return int(a.item())


class _Transposed:
    """W^T view (geometry.py:215 ``w.T``; solvers.py:111 ``w.T.tocsr()``)."""

    def __init__(self, w: LineProjector):
        self._w = w
        self.shape = (w.shape[1], w.shape[0])

    @property
    def T(self):
        return self._w

    def tocsr(self):
        return self

    def __matmul__(self, v):
        return self._w.backward(v)

    def dot(self, v):
        return self._w.backward(v)

    def sum(self, axis=None):
        if axis in (0, -2):
            return self._w.sum(axis=1)
        if axis in (1, -1):
            return self._w.sum(axis=0)
        return self._w.sum(axis)


def build_projector(g: Geometry, kernel: str = "line", precision: str = "float64",
                    mode: str | None = None, device=None) -> LineProjector:
    """Matrix-free projector (geometry.py:178-197): ``kernel="line"`` (exact
    intersection lengths, every mode) or ``"joseph"`` (two-pixel interpolation
    per slab, geometry.py:131-175; float64 parity mode only)."""
    if kernel not in ("line", "joseph"):
        raise ValueError(f"unknown kernel '{kernel}'")
    if kernel == "joseph" and (precision != "float64" or mode not in (None, "parity")):
        raise ValueError("kernel='joseph' is implemented in float64 parity mode only")
    return LineProjector(g, precision=precision, mode=mode, device=device, kernel=kernel)


def apply(w, x):
    """Forward projection W x (geometry.py:200-206)."""
    n = x.numel() if D.is_torch(x) else np.asarray(x).shape[0]
    if n != w.shape[1]:
        raise DimensionMismatchError(f"apply: vector length {n} != n_cols {w.shape[1]}")
    return w @ x


def apply_transpose(w, y):
    """Backprojection W^T y (geometry.py:209-215)."""
    n = y.numel() if D.is_torch(y) else np.asarray(y).shape[0]
    if n != w.shape[0]:
        raise DimensionMismatchError(
            f"apply_transpose: vector length {n} != n_rows {w.shape[0]}")
    return w.T @ y
