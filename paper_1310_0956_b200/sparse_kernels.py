"""Error types and the dense coarse-level factorization, on the GPU.

Mirrors /root/reference/pkg/src/wmgtomo/sparse_kernels.py:
  * ``DimensionMismatchError`` / ``NotPositiveDefiniteError`` (:22-27),
  * ``DenseFactorization`` / ``cholesky_factor`` / ``cholesky_solve`` (:42-75),
    here holding a float64 lower factor in HBM, factored and solved by the
    hand-written ``wmg_cholesky_factor`` / ``wmg_cholesky_solve`` kernels
    (csrc/cholesky.cu: blocked potrf with DMMA panel/update, blocked potrs),
  * ``spd_inverse_``: the WMG leaves' batched SPD inverse on the fp64 tensor
    cores (hand-written DMMA sweep, ``wmg_spd_inverse``).
``spgemm`` / ``seeded_uniform`` are not on the B200 path (the hierarchy is
matrix-free, inputs are generated host-side) -- SURVEY.md s2 row 4.
"""
from __future__ import annotations

SPGEMM_DROP_TOL = 1e-15


class DimensionMismatchError(ValueError):
    """Operands have incompatible shapes."""


class NotPositiveDefiniteError(ValueError):
    """A matrix expected to be symmetric positive definite is not."""


class DenseFactorization:
    """Lower Cholesky factor(s) of SPD matrices resident on the GPU.

    ``lower`` is a torch float64 tensor of shape (dim, dim) or (batch, dim, dim)
    (reference field, sparse_kernels.py:40-45).  ``inverse`` (optional) holds
    G^-1 for the WMG coarse solves: one bandwidth-bound GEMV per solve instead
    of two latency-bound triangular solves (same kappa * eps forward-error
    class).  When the inverse came from ``spd_inverse_`` (no Cholesky at setup)
    the factor is computed on first access from the kept ``gram`` copy.
    Immutable like the reference's frozen dataclass.
    """

    __slots__ = ("dimension", "_lower", "_inv", "_gram", "_padded", "_np")

    def __init__(self, dimension: int, lower=None, inverse=None, gram=None, padded=None,
                 was_numpy=False):
        object.__setattr__(self, "dimension", dimension)
        object.__setattr__(self, "_lower", lower)
        object.__setattr__(self, "_inv", inverse)   # dense tensor or PackedSymmetric
        object.__setattr__(self, "_gram", gram)
        # (padded factor (b, q, q), diagonal-block inverses, q) of wmg_cholesky_factor
        object.__setattr__(self, "_padded", padded)
        object.__setattr__(self, "_np", bool(was_numpy))

    @property
    def inverse(self):
        """G^-1 as a dense (dim, dim) tensor (unpacked on access when stored
        packed; the coarse solves use the packed form directly)."""
        if isinstance(self._inv, PackedSymmetric):
            return self._inv.dense()[0]
        return self._inv

    def __setattr__(self, name, value):
        raise AttributeError("DenseFactorization is immutable")

    def __repr__(self):
        return f"DenseFactorization(dimension={self.dimension})"

    def _ensure_factor(self):
        """Factor the kept Gram on first use (leaves built by spd_inverse_)."""
        if self._padded is None and self._gram is not None:
            g = self._gram
            gl = g.tril()
            full = gl + gl.tril(-1).transpose(-1, -2)
            f = cholesky_factor(full)
            object.__setattr__(self, "_lower", f._lower)
            object.__setattr__(self, "_padded", f._padded)
        if self._padded is None and self._lower is not None:
            raise ValueError("factorization has no device factor")

    @property
    def lower(self):
        """The lower Cholesky factor (zeros above the diagonal), in the caller's
        array type (numpy when the factored matrix was numpy)."""
        if self._lower is None:
            self._ensure_factor()
        low = self._lower
        if low is not None and self._np:
            return low.cpu().numpy()
        return low

    def solve(self, rhs):
        return cholesky_solve(self, rhs)

    def apply_inverse(self, rhs, out=None):
        """G^-1 rhs via the stored inverse: our batched GEMV kernel (falls back to
        the triangular solves when no inverse is stored)."""
        if self._inv is None:
            return cholesky_solve(self, rhs)
        return batched_gemv(self._inv, rhs, out)


def spd_inverse_(g, names=None):
    """In-place inverse of SPD matrices g ((p,p) or (b,p,p) float64 CUDA,
    row-major; only the lower triangle is read) with the hand-written DMMA sweep
    (``wmg_spd_inverse``): on return g holds the full symmetric inverse.

    Replaces potrf + cho_solve of the reference (sparse_kernels.py:53-75) for the
    WMG leaves.  Orders that are not a multiple of 128 go through an identity-
    padded copy.  Raises NotPositiveDefiniteError naming the first failing
    matrix (``names[i]``) and its leading minor, like potrf's info."""
    import ctypes
    import torch
    from . import _native as N
    g3 = g if g.dim() == 3 else g.unsqueeze(0)
    if g3.shape[-1] != g3.shape[-2]:
        raise DimensionMismatchError(f"spd_inverse_: matrix is not square {tuple(g.shape)}")
    if not (g3.is_cuda and g3.dtype == torch.float64 and g3.is_contiguous()):
        raise ValueError("spd_inverse_: expects contiguous float64 CUDA matrices")
    b, p = g3.shape[0], g3.shape[-1]
    if b == 0 or p == 0:
        return g
    q = -(-p // 128) * 128
    work_mat = g3
    if q != p:
        work_mat = torch.zeros((b, q, q), dtype=torch.float64, device=g.device)
        work_mat[:, :p, :p].copy_(g3)
        work_mat.diagonal(dim1=1, dim2=2)[:, p:].fill_(1.0)
    nbytes = ctypes.c_size_t()
    N.call("wmg_spd_inverse_workspace", b, q, ctypes.byref(nbytes))
    work = torch.empty(nbytes.value // 8, dtype=torch.float64, device=g.device)
    info = torch.empty(b, dtype=torch.int32, device=g.device)
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    N.call("wmg_spd_inverse", b, q, ctypes.c_void_p(work_mat.data_ptr()), q * q,
           ctypes.c_void_p(info.data_ptr()), ctypes.c_void_p(work.data_ptr()), st)
    bad = info.cpu().numpy()
    for i, code in enumerate(bad):
        if 0 < code <= p:
            name = names[i] if names is not None else f"matrix {i}"
            raise NotPositiveDefiniteError(
                f"{name}: leading minor of order {int(code)} is not positive definite")
    if q != p:
        g3.copy_(work_mat[:, :p, :p])
    return g


class PackedSymmetric:
    """Symmetric float64 matrices (p % 128 == 0) stored as their lower 128 x 128
    tiles (``wmg_sym_pack`` layout): half the bytes of the dense storage.  The
    WMG leaf inverses live in this form; ``batched_gemv`` on it runs
    ``wmg_packed_symv`` (every tile read once, fixed-order partial sums).
    Indexing with a slice selects matrices (a view); ``dense()`` unpacks."""

    def __init__(self, data, p: int):
        self.data = data            # (batch, elems) float64, contiguous rows
        self.p = int(p)

    @classmethod
    def pack(cls, full):
        """Pack full symmetric (b, p, p) (or (p, p)) CUDA float64 matrices."""
        import ctypes
        import torch
        from . import _native as N
        f3 = full if full.dim() == 3 else full.unsqueeze(0)
        b, p = f3.shape[0], f3.shape[-1]
        elems = ctypes.c_longlong()
        N.call("wmg_packed_sym_sizes", b, p, ctypes.byref(elems), None)
        data = torch.empty((b, elems.value), dtype=torch.float64, device=full.device)
        st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        N.call("wmg_sym_pack", b, p, ctypes.c_void_p(f3.data_ptr()), p * p,
               ctypes.c_void_p(data.data_ptr()), elems.value, st)
        return cls(data, p)

    @property
    def shape(self):
        return (self.data.shape[0], self.p, self.p)

    def __len__(self):
        return self.data.shape[0]

    def __getitem__(self, idx):
        if isinstance(idx, slice):
            return PackedSymmetric(self.data[idx], self.p)
        return PackedSymmetric(self.data[idx:idx + 1], self.p)

    def dense(self):
        """(b, p, p) full matrices (API / tests; not on the hot path)."""
        import torch
        T = 128
        nt = self.p // T
        b = self.data.shape[0]
        tiles = self.data.view(b, -1, T, T)
        out = torch.empty((b, self.p, self.p), dtype=torch.float64, device=self.data.device)
        t = 0
        for i in range(nt):
            for j in range(i + 1):
                blk = tiles[:, t]
                out[:, i * T:(i + 1) * T, j * T:(j + 1) * T] = blk
                if i != j:
                    out[:, j * T:(j + 1) * T, i * T:(i + 1) * T] = blk.transpose(1, 2)
                t += 1
        return out

    def gemv(self, x, out=None):
        import ctypes
        import torch
        from . import _native as N
        x2 = x if x.dim() == 2 else x.unsqueeze(0)
        b, p = self.data.shape[0], self.p
        if tuple(x2.shape) != (b, p):
            raise DimensionMismatchError(f"packed symv: rhs {tuple(x.shape)} vs {self.shape}")
        x2 = x2.contiguous()
        y = torch.empty((b, p), dtype=torch.float64, device=x.device) if out is None else out
        nbytes = ctypes.c_size_t()
        N.call("wmg_packed_sym_sizes", b, p, None, ctypes.byref(nbytes))
        scratch = torch.empty(nbytes.value // 8, dtype=torch.float64, device=x.device)
        st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        N.call("wmg_packed_symv", b, p, ctypes.c_void_p(self.data.data_ptr()),
               self.data.stride(0), ctypes.c_void_p(x2.data_ptr()), p,
               ctypes.c_void_p(y.data_ptr()), p, ctypes.c_void_p(scratch.data_ptr()), st)
        return y if x.dim() == 2 else y.view(p)


def batched_gemv(A, x, out=None):
    """y_b = A_b x_b (A: (p,p) or (b,p,p) float64 CUDA, or PackedSymmetric;
    x: (p,) or (b,p))."""
    import ctypes
    import torch
    from . import _native as N
    if isinstance(A, PackedSymmetric):
        return A.gemv(x, out)
    A3 = A if A.dim() == 3 else A.unsqueeze(0)
    x2 = x if x.dim() == 2 else x.unsqueeze(0)
    b, p = A3.shape[0], A3.shape[-1]
    if tuple(x2.shape) != (b, p):
        raise DimensionMismatchError(f"batched_gemv: rhs {tuple(x.shape)} vs {tuple(A.shape)}")
    if not A3.is_contiguous():
        raise ValueError("batched_gemv: matrices must be row-major contiguous")
    x2 = x2.contiguous()
    y = torch.empty((b, p), dtype=torch.float64, device=x.device) if out is None else out
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    N.call("wmg_batched_gemv", b, p, ctypes.c_void_p(A3.data_ptr()), p * p,
           ctypes.c_void_p(x2.data_ptr()), p, ctypes.c_void_p(y.data_ptr()), p, st)
    return y if x.dim() == 2 else y.view(p)


def _pad_order(p: int) -> int:
    return -(-p // 128) * 128


def cholesky_factor(g, sym_tol: float = 1e-10) -> DenseFactorization:
    """Factor dense SPD matrices: numpy or torch, (d, d) or (b, d, d).

    Same contract as the reference (sparse_kernels.py:53-65): non-square ->
    DimensionMismatchError; asymmetric beyond sym_tol * max|G| or not positive
    definite -> NotPositiveDefiniteError.  The factorization runs on the GPU
    (``wmg_cholesky_factor``: blocked potrf, DMMA panel and trailing update);
    orders that are not a multiple of 128 are factored through an identity-
    padded copy.  ``lower`` is returned in the caller's array type.
    """
    import ctypes

    import torch

    from . import _device as D
    from . import _native as N
    was_np = not isinstance(g, torch.Tensor)
    if was_np:
        import numpy as np
        ga = np.asarray(g, dtype=np.float64)
        if ga.ndim not in (2, 3) or ga.shape[-1] != ga.shape[-2]:
            raise DimensionMismatchError(f"cholesky_factor: matrix is not square {ga.shape}")
        D.require_cuda()
        g = torch.from_numpy(np.ascontiguousarray(ga)).cuda()
    else:
        if g.dim() not in (2, 3) or g.shape[-1] != g.shape[-2]:
            raise DimensionMismatchError(
                f"cholesky_factor: matrix is not square {tuple(g.shape)}")
        D.require_cuda()
        g = g.to(device="cuda" if not g.is_cuda else g.device, dtype=torch.float64)
    if g.numel():
        scale = g.abs().amax()
        asym = (g - g.transpose(-1, -2)).abs().amax()
        if float(scale) and float(asym) > sym_tol * float(scale):
            raise NotPositiveDefiniteError("matrix is not symmetric")
    g3 = g if g.dim() == 3 else g.unsqueeze(0)
    b, p = g3.shape[0], g3.shape[-1]
    if p == 0 or b == 0:
        return DenseFactorization(dimension=p, lower=g.clone(), was_numpy=was_np)
    q = _pad_order(p)
    work = torch.zeros((b, q, q), dtype=torch.float64, device=g.device)
    work[:, :p, :p].copy_(g3)
    if q != p:
        work.diagonal(dim1=1, dim2=2)[:, p:].fill_(1.0)
    elems = ctypes.c_longlong()
    N.call("wmg_cholesky_dinv_elems", q, ctypes.byref(elems))
    dinv = torch.empty((b, elems.value), dtype=torch.float64, device=g.device)
    info = torch.empty(b, dtype=torch.int32, device=g.device)
    N.call("wmg_cholesky_factor", b, q, D.ptr(work), q * q, D.ptr(dinv), D.ptr(info),
           D.stream_handle())
    bad = info.cpu()
    if int(bad.max()) > 0:
        i = int(bad.argmax())
        where = f"matrix {i}: " if b > 1 else ""
        raise NotPositiveDefiniteError(
            f"{where}leading minor of order {int(bad[i])} is not positive definite")
    lower = work[:, :p, :p] if q != p else work
    if g.dim() == 2:
        lower = lower[0]
    return DenseFactorization(dimension=p, lower=lower, padded=(work, dinv, q),
                              was_numpy=was_np)


def cholesky_solve(f: DenseFactorization, rhs):
    """Solve L L^T z = rhs on the device (``wmg_cholesky_solve``: blocked
    forward / backward substitution, fixed summation order); rhs (d,), (d, k)
    -- the reference's shapes (sparse_kernels.py:68-75) -- or, for batched
    factors, (b, d) / (b, d, k).  Returns the caller's array type."""
    import torch

    from . import _device as D
    from . import _native as N
    was_np = not isinstance(rhs, torch.Tensor)
    r = torch.as_tensor(rhs, dtype=torch.float64) if was_np else rhs.to(torch.float64)
    p = f.dimension
    pk = f._padded
    batched = pk is not None and pk[0].shape[0] > 1 or (f._lower is not None and
                                                          f._lower.dim() == 3)
    if batched:
        ok = r.dim() in (2, 3) and r.shape[1] == p
    else:
        ok = r.dim() in (1, 2) and r.shape[0] == p
    if not ok:
        raise DimensionMismatchError(
            f"cholesky_solve: rhs shape {tuple(r.shape)} does not match dimension {p}")
    if pk is None:
        f._ensure_factor()
        pk = f._padded
    work, dinv, q = pk
    b = work.shape[0]
    dev = work.device
    r3 = r.reshape(b, p, -1) if batched else r.reshape(1, p, -1)
    k = r3.shape[-1]
    B = torch.zeros((b, q, k), dtype=torch.float64, device=dev)
    B[:, :p, :].copy_(r3)
    if k and p:
        N.call("wmg_cholesky_solve", b, q, D.ptr(work), q * q, D.ptr(dinv), D.ptr(B), q * k, k,
               D.stream_handle())
    out = B[:, :p, :].reshape(r.shape)
    if was_np:
        return out.cpu().numpy()
    return out.to(r.device) if r.device != dev else out
