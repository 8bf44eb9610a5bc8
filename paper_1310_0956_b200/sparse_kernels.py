"""Error types and the dense coarse-level factorization, on the GPU.

Mirrors /root/reference/pkg/src/wmgtomo/sparse_kernels.py:
  * ``DimensionMismatchError`` / ``NotPositiveDefiniteError`` (:22-27),
  * ``DenseFactorization`` / ``cholesky_factor`` / ``cholesky_solve`` (:42-75),
    here holding a float64 lower factor in HBM (cuSOLVER potrf through torch)
    and solving with two triangular solves on the device.
``spgemm`` / ``seeded_uniform`` are not on the B200 path (the hierarchy is
matrix-free, inputs are generated host-side) -- SURVEY.md s2 row 4.
"""
from __future__ import annotations

from dataclasses import dataclass

SPGEMM_DROP_TOL = 1e-15


class DimensionMismatchError(ValueError):
    """Operands have incompatible shapes."""


class NotPositiveDefiniteError(ValueError):
    """A matrix expected to be symmetric positive definite is not."""


@dataclass(frozen=True)
class DenseFactorization:
    """Lower Cholesky factor(s) of SPD matrices resident on the GPU.

    ``lower`` is a torch float64 tensor of shape (dim, dim) or (batch, dim, dim).
    ``inverse`` (optional) holds G^-1 = L^-T L^-1 for the WMG coarse solves: one
    bandwidth-bound GEMV per solve instead of two latency-bound triangular
    solves (same kappa * eps forward-error class).
    """

    dimension: int
    lower: object
    inverse: object = None

    def solve(self, rhs):
        return cholesky_solve(self, rhs)

    def apply_inverse(self, rhs, out=None):
        """G^-1 rhs via the stored inverse: our batched GEMV kernel (falls back to
        the triangular solves when no inverse is stored)."""
        if self.inverse is None:
            return cholesky_solve(self, rhs)
        return batched_gemv(self.inverse, rhs, out)


def batched_gemv(A, x, out=None):
    """y_b = A_b x_b (A: (p,p) or (b,p,p) float64 CUDA, x: (p,) or (b,p))."""
    import ctypes
    import torch
    from . import _native as N
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


def cholesky_factor(g, sym_tol: float = 1e-10) -> DenseFactorization:
    """Factor dense SPD matrices (torch CUDA tensor, (d,d) or (b,d,d)).

    Same contract as the reference (sparse_kernels.py:53-65): non-square ->
    DimensionMismatchError; asymmetric beyond sym_tol * max|G| or not positive
    definite -> NotPositiveDefiniteError.
    """
    import torch

    g = torch.as_tensor(g)
    if g.dim() not in (2, 3) or g.shape[-1] != g.shape[-2]:
        raise DimensionMismatchError(f"cholesky_factor: matrix is not square {tuple(g.shape)}")
    if not g.is_cuda:
        raise RuntimeError("cholesky_factor: expects a CUDA tensor (no CPU fallback)")
    g = g.to(torch.float64)
    if g.numel():
        scale = g.abs().amax()
        asym = (g - g.transpose(-1, -2)).abs().amax()
        if float(scale) and float(asym) > sym_tol * float(scale):
            raise NotPositiveDefiniteError("matrix is not symmetric")
    lower, info = torch.linalg.cholesky_ex(g)
    bad = int(info.max()) if info.numel() else 0
    if bad > 0:
        raise NotPositiveDefiniteError(
            f"leading minor of order {bad} is not positive definite")
    return DenseFactorization(dimension=int(g.shape[-1]), lower=lower)


def cholesky_solve(f: DenseFactorization, rhs):
    """Solve L L^T z = rhs on the device; rhs (d,), (d,k), (b,d) or (b,d,k)."""
    import torch

    rhs = torch.as_tensor(rhs)
    if rhs.shape[-1] != f.dimension and (rhs.dim() < 2 or rhs.shape[-2] != f.dimension):
        raise DimensionMismatchError(
            f"cholesky_solve: rhs length {rhs.shape[-1]} != dimension {f.dimension}")
    L = f.lower
    if L.dim() == 2:
        if rhs.dim() == 1:
            return torch.cholesky_solve(rhs.unsqueeze(1), L).squeeze(1)
        return torch.cholesky_solve(rhs, L)
    # batched factors: rhs (b, d) or (b, d, k)
    if rhs.dim() == 2:
        return torch.cholesky_solve(rhs.unsqueeze(2), L).squeeze(2)
    return torch.cholesky_solve(rhs, L)
