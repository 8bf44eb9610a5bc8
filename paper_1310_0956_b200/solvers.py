"""SIRT, normal operator, BiCGStab, CGLS / WMG-CGLS and GMRES on the GPU.

Drop-in for /root/reference/pkg/src/wmgtomo/solvers.py: same ``SolverConfig``
(:27-37), ``ConvergenceRecord`` (:41-60), ``find_kopt`` (:63-68), status strings
(:22-24), breakdown constant (:20), ``sirt_scaling`` (:79-86), ``sirt_solve``
(:95-137), ``normal_operator`` (:140-156) and ``bicgstab_solve`` (:159-243)
semantics.  Every vector lives in HBM; every vector op is one of our sm_100a
kernels.  Host code only sequences kernels and reads back the O(1) scalars the
reference needs per iteration (breakdown tests, logging, tolerance stop).

Reductions use the deterministic DET_SUM (csrc/vecops.cu), so each solver is
bit-reproducible and bit-identical to its restatement in ``oracle/solvers.py``.
Against the reference itself: ``sirt_solve`` is bit-identical in x (elementwise
ops + the parity projector; only the logged norms use a different summation
order), the Krylov solvers agree within the reference's own reordering envelope
(SURVEY.md s0.5).

New solvers (not in the reference): ``cgls_solve``
(textbook CGLS; with ``precond`` the flexible Polak-Ribiere PCG on the normal
equations -- "WMG-CGLS") and ``gmres_solve`` (right-preconditioned restarted
GMRES with classical Gram-Schmidt + reorthogonalisation).  Both log the
normal-equations residual ||W^T(b - W x) - lam x|| / ||W^T b - ...||.
"""
from __future__ import annotations

import time
import weakref
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import _device as D
from . import _native as N
from .sparse_kernels import DimensionMismatchError

BREAKDOWN_REL_TOL = 1e-14

STATUS_CONVERGED = "converged"
STATUS_MAX_ITERATIONS = "max-iterations"
STATUS_BREAKDOWN = "breakdown"


@dataclass
class SolverConfig:
    max_iterations: int = 100
    residual_tolerance: float = 0.0
    regularization_lambda: float = 0.0

    def __post_init__(self):
        if self.max_iterations < 1:
            raise ValueError("max_iterations must be >= 1")
        if self.residual_tolerance < 0 or self.regularization_lambda < 0:
            raise ValueError("tolerance and lambda must be nonnegative")


@dataclass
class ConvergenceRecord:
    """Per-iteration (index, rel. residual, rel. L2 error, rel. Linf error, seconds)."""

    iterations: list = field(default_factory=list)
    rel_residual: list = field(default_factory=list)
    rel_err_l2: list = field(default_factory=list)
    rel_err_linf: list = field(default_factory=list)
    seconds: list = field(default_factory=list)
    status: str = STATUS_MAX_ITERATIONS

    def log(self, k, rel_res, err2, errinf, secs):
        self.iterations.append(int(k))
        self.rel_residual.append(float(rel_res))
        self.rel_err_l2.append(None if err2 is None else float(err2))
        self.rel_err_linf.append(None if errinf is None else float(errinf))
        self.seconds.append(float(secs))

    @property
    def has_errors(self) -> bool:
        return all(e is not None for e in self.rel_err_l2) and bool(self.rel_err_l2)


def find_kopt(record: ConvergenceRecord) -> int:
    """First iteration index attaining the minimum relative L2 error."""
    if not record.has_errors:
        raise ValueError("record has no error data; solve with x_ex provided")
    errs = np.asarray(record.rel_err_l2, dtype=np.float64)
    return int(record.iterations[int(np.argmin(errs))])


@dataclass(frozen=True)
class SirtScaling:
    """Inverse column sums (c, length N) and inverse row sums (r, length M) of W.

    ``c`` / ``r`` are numpy arrays (reference contract); ``c_dev`` / ``r_dev``
    are the same values resident in HBM.
    """

    c: np.ndarray
    r: np.ndarray
    c_dev: object = field(default=None, repr=False, compare=False)
    r_dev: object = field(default=None, repr=False, compare=False)


def sirt_scaling(w) -> SirtScaling:
    """r = 1/rowsum(W), c = 1/colsum(W), zero sums -> 0 (solvers.py:79-86)."""
    t = D.require_cuda()
    rows = w.row_sums_dev()
    cols = w.col_sums_dev()
    r = t.empty_like(rows)
    c = t.empty_like(cols)
    D.recip(r, rows)
    D.recip(c, cols)
    return SirtScaling(c=c.cpu().numpy(), r=r.cpu().numpy(), c_dev=c, r_dev=r)


def _device_scaling(w, scaling):
    if scaling is None:
        scaling = sirt_scaling(w)
    if scaling.c_dev is None:
        c, _ = D.to_device(scaling.c)
        r, _ = D.to_device(scaling.r)
        return c, r
    return scaling.c_dev, scaling.r_dev


class _ErrorTracker:
    """error_metrics (phantom.py:64-75) evaluated on the device each iteration."""

    def __init__(self, x_ex, n, device):
        self.active = x_ex is not None
        if not self.active:
            return
        t = D.torch()
        xe, _ = D.to_device(x_ex)
        if xe.numel() != n:
            raise ValueError("error_metrics: length mismatch")
        self.x_ex = xe
        nrm = D.det_reduce([(N.RED_SQ, xe, None, None)])
        inf = D.maxabs(xe)
        vals = t.cat([nrm, inf]).cpu().numpy()
        self.norm2 = float(np.sqrt(vals[0]))
        self.norminf = float(vals[1])
        if self.norm2 == 0.0:
            raise ValueError("error_metrics: exact image is identically zero")

    def device_terms(self, x):
        """[sum (x - x_ex)^2, max |x - x_ex|] on the device (no sync)."""
        if not self.active:
            return None
        return D.error_metrics_dev(x, self.x_ex)

    def finish(self, host_terms):
        if not self.active:
            return None, None
        return (float(np.sqrt(host_terms[0]) / self.norm2),
                float(host_terms[1] / self.norminf))


def _sino(w, t):
    """Sinogram-space reduction hook: allreduce partials when W is angle-sharded."""
    red = getattr(w, "reduce_sino_", None)
    return red(t) if red is not None else t


def _readback(*tensors):
    """One D2H copy for several small device tensors -> numpy float64."""
    t = D.torch()
    parts = [x.reshape(-1) for x in tensors if x is not None]
    return t.cat(parts).cpu().numpy() if parts else np.zeros(0)


# --------------------------------------------------------------------- SIRT
def sirt_solve(w, b, x0, cfg: SolverConfig, x_ex=None, scaling: Optional[SirtScaling] = None):
    """Gregor-Benson scaled SIRT: x <- x + C W^T R (b - W x) - lambda C x.

    Same iterate sequence as solvers.py:95-137 (bit-identical x with the
    float64 parity projector); the logged norms use DET_SUM.
    """
    t = D.require_cuda()
    M, Nn = w.shape
    bd, was_np = D.to_device(b)
    if x0 is None:
        x = t.zeros(Nn, dtype=t.float64, device=bd.device)
    else:
        x0d, _ = D.to_device(x0)
        x = x0d.clone()
    if bd.numel() != M or x.numel() != Nn:
        raise DimensionMismatchError("sirt_solve: dimension mismatch")
    c, r = _device_scaling(w, scaling)
    lam = cfg.regularization_lambda
    errs = _ErrorTracker(x_ex, Nn, bd.device)

    record = ConvergenceRecord()
    t0 = time.perf_counter()
    wx = t.empty(M, dtype=t.float64, device=bd.device)
    res = t.empty(M, dtype=t.float64, device=bd.device)
    tmp = t.empty(M, dtype=t.float64, device=bd.device)
    g = t.empty(Nn, dtype=t.float64, device=bd.device)
    w.forward_(x, wx)
    D.axpy(res, bd, 1.0, -1, wx)                      # res = b - W x
    h = _readback(_sino(w, D.det_norm_sq(res)), errs.device_terms(x))
    res_norm0 = float(np.sqrt(h[0]))
    e2, einf = errs.finish(h[1:3]) if errs.active else (None, None)
    record.log(0, 1.0, e2, einf, time.perf_counter() - t0)
    if res_norm0 == 0.0:
        record.status = STATUS_CONVERGED
        return D.to_caller(x, was_np), record

    for k in range(1, cfg.max_iterations + 1):
        D.hadamard(tmp, r, res)                       # r * res
        w.backward_(tmp, g)                           # W^T (r * res)
        N.call("wmg_sirt_update", Nn, D.ptr(x), D.ptr(c), D.ptr(g), float(lam),
               D.stream_handle())
        w.forward_(x, wx)
        D.axpy(res, bd, 1.0, -1, wx)
        h = _readback(_sino(w, D.det_norm_sq(res)), errs.device_terms(x))
        rel = float(np.sqrt(h[0])) / res_norm0
        e2, einf = errs.finish(h[1:3]) if errs.active else (None, None)
        record.log(k, rel, e2, einf, time.perf_counter() - t0)
        if cfg.residual_tolerance > 0 and rel < cfg.residual_tolerance:
            record.status = STATUS_CONVERGED
            return D.to_caller(x, was_np), record
    record.status = STATUS_MAX_ITERATIONS
    return D.to_caller(x, was_np), record


# --------------------------------------------------------- normal operator
class NormalOperator:
    """v -> W^T (W v) + lambda v without forming W^T W (solvers.py:140-156).

    Callable on numpy (returns numpy) or CUDA tensors (stays on device).
    """

    _wmg_device = True

    def __init__(self, w, lam: float):
        if lam < 0:
            raise ValueError("lambda must be nonnegative")
        self.w = w
        self.lam = float(lam)
        self.shape = (w.shape[1], w.shape[1])
        self._tmp = None

    def apply_(self, v, out):
        t = D.torch()
        if v.numel() != self.w.shape[1]:
            raise DimensionMismatchError(
                f"normal_operator: length {v.numel()} != {self.w.shape[1]}")
        if self._tmp is None or self._tmp.device != v.device:
            self._tmp = t.empty(self.w.shape[0], dtype=t.float64, device=v.device)
        self.w.forward_(v, self._tmp)
        self.w.backward_(self._tmp, out)
        if self.lam != 0:
            D.add_scaled(out, out, self.lam, +1, v)
        return out

    def __call__(self, v):
        t = D.torch()
        vd, was_np = D.to_device(v)
        if vd.numel() != self.w.shape[1]:
            raise DimensionMismatchError(
                f"normal_operator: length {vd.numel()} != {self.w.shape[1]}")
        out = t.empty(self.w.shape[1], dtype=t.float64, device=vd.device)
        self.apply_(vd, out)
        return D.to_caller(out, was_np)


def normal_operator(w, lam: float) -> Callable:
    return NormalOperator(w, lam)


def _as_device_op(fn):
    """Wrap a callable so it maps CUDA float64 tensors to CUDA float64 tensors.

    Our own operators (``_wmg_device``) run on the GPU directly; a user callable
    written for numpy is bridged (host round trip for that callable only).
    """
    if fn is None:
        return None
    if getattr(fn, "_wmg_device", False):
        if hasattr(fn, "apply_"):
            t = D.torch()

            def dev(v):
                out = t.empty_like(v)
                return fn.apply_(v, out)
            return dev
        return fn

    def bridged(v):
        t = D.torch()
        res = fn(v.detach().cpu().numpy())
        return t.as_tensor(np.asarray(res, dtype=np.float64), device=v.device)
    return bridged


# ----------------------------------------------------------------- BiCGStab
def bicgstab_solve(op, f, precond=None, x0=None, cfg: SolverConfig = None, x_ex=None):
    """Van der Vorst BiCGStab with right preconditioning (solvers.py:159-243)."""
    t = D.require_cuda()
    if cfg is None:
        cfg = SolverConfig()
    fd, was_np = D.to_device(f)
    n = fd.numel()
    if x0 is None:
        x = t.zeros_like(fd)
    else:
        x = D.to_device(x0)[0].clone()
    if x.shape != fd.shape:
        raise DimensionMismatchError("bicgstab_solve: x0/f length mismatch")
    A = _as_device_op(op)
    minv = (lambda v: v) if precond is None else _as_device_op(precond)
    errs = _ErrorTracker(x_ex, n, fd.device)
    record = ConvergenceRecord()
    t0 = time.perf_counter()
    r = t.empty_like(fd)
    D.axpy(r, fd, 1.0, -1, A(x))                      # r = f - op(x)
    h = _readback(D.det_norm_sq(r), errs.device_terms(x))
    res_norm0 = float(np.sqrt(h[0]))
    e2, einf = errs.finish(h[1:3]) if errs.active else (None, None)
    record.log(0, 1.0, e2, einf, time.perf_counter() - t0)
    if res_norm0 == 0.0:
        record.status = STATUS_CONVERGED
        return D.to_caller(x, was_np), record

    r_hat = r.clone()
    r_hat_norm = res_norm0
    rho_prev = alpha = omega = 1.0
    v = t.zeros_like(r)
    p = t.zeros_like(r)
    s = t.empty_like(r)
    r_norm = res_norm0
    for k in range(1, cfg.max_iterations + 1):
        rho = float(_readback(D.det_dot(r_hat, r))[0])
        if abs(rho) <= BREAKDOWN_REL_TOL * r_hat_norm * r_norm:
            record.status = STATUS_BREAKDOWN
            return D.to_caller(x, was_np), record
        if k == 1:
            p.copy_(r)
        else:
            beta = (rho / rho_prev) * (alpha / omega)
            N.call("wmg_bicg_p", n, D.ptr(p), D.ptr(r), beta, omega, D.ptr(v),
                   D.stream_handle())
        p_hat = minv(p)
        v = A(p_hat)
        hv = _readback(D.det_reduce([(N.RED_DOT, r_hat, v, None), (N.RED_SQ, v, None, None)]))
        denom, v_norm = float(hv[0]), float(np.sqrt(hv[1]))
        if abs(denom) <= BREAKDOWN_REL_TOL * r_hat_norm * v_norm:
            record.status = STATUS_BREAKDOWN
            return D.to_caller(x, was_np), record
        alpha = rho / denom
        D.axpy(s, r, alpha, -1, v)                    # s = r - alpha v
        s_hat = minv(s)
        tt_vec = A(s_hat)
        ht = _readback(D.det_reduce([(N.RED_SQ, tt_vec, None, None),
                                     (N.RED_DOT, tt_vec, s, None)]))
        tt, ts = float(ht[0]), float(ht[1])
        if tt < BREAKDOWN_REL_TOL ** 2 * res_norm0 ** 2:
            D.axpy(x, x, alpha, +1, p_hat)
            r = s.clone()
            h = _readback(D.det_norm_sq(r), errs.device_terms(x))
            rel = float(np.sqrt(h[0])) / res_norm0
            e2, einf = errs.finish(h[1:3]) if errs.active else (None, None)
            record.log(k, rel, e2, einf, time.perf_counter() - t0)
            record.status = STATUS_CONVERGED
            return D.to_caller(x, was_np), record
        omega = ts / tt
        N.call("wmg_bicg_x", n, D.ptr(x), alpha, D.ptr(p_hat), omega, D.ptr(s_hat),
               D.stream_handle())
        D.axpy(r, s, omega, -1, tt_vec)               # r = s - omega t
        rho_prev = rho
        h = _readback(D.det_norm_sq(r), errs.device_terms(x))
        r_norm = float(np.sqrt(h[0]))
        rel = r_norm / res_norm0
        e2, einf = errs.finish(h[1:3]) if errs.active else (None, None)
        record.log(k, rel, e2, einf, time.perf_counter() - t0)
        if cfg.residual_tolerance > 0 and rel < cfg.residual_tolerance:
            record.status = STATUS_CONVERGED
            return D.to_caller(x, was_np), record
        if abs(omega) < BREAKDOWN_REL_TOL:
            record.status = STATUS_BREAKDOWN
            return D.to_caller(x, was_np), record
    record.status = STATUS_MAX_ITERATIONS
    return D.to_caller(x, was_np), record


FUSED_CGLS = True      # tests switch it off to compare with the unfused kernels


class _GraphedLoop:
    """Runs a device-only loop body: eagerly once (warm-up), then captured once
    as a CUDA graph and replayed for every further iteration."""

    def __init__(self, body, tolerate_capture_failure=False):
        self.body = body
        self.calls = 0
        self.graph = None
        self.eager = False
        self.tolerant = tolerate_capture_failure

    def step(self):
        t = D.torch()
        self.calls += 1
        if self.calls == 1 or self.eager:
            self.body()
            return
        if self.graph is None:
            try:
                self.graph, _ = D.capture_graph(self.body, t.cuda.current_device())
            except RuntimeError as exc:
                if not self.tolerant:
                    raise
                # sharded loop whose collectives could not be captured: this rank
                # keeps issuing the same sequence eagerly
                import warnings
                warnings.warn(f"sharded iteration not captured, running eagerly: {exc}")
                self.eager = True
                self.body()
                return
        self.graph.replay()


def _graphable(w, precond):
    # sharded: the loop holds collectives; NCCL's are stream-ordered and are
    # captured with the kernels, host-side ones (gloo) keep the loop eager
    if not getattr(w, "graph_capturable", getattr(w, "world", 1) == 1):
        return False
    if not (hasattr(w, "forward_") and hasattr(w, "backward_")):
        return False
    return precond is None or hasattr(precond, "_eager")


def _cgls_graphed(w, bd, x, lam, precond, cfg, errs, was_np, record, t0):
    """CGLS / flexible PCG-NE with device-resident scalars: one graph replay and
    one 12-double D2H per iteration; same arithmetic as the eager path (see
    cgls_solve), hence bit-identical iterates and records."""
    t = D.torch()
    dev = bd.device
    M_, Nn = w.shape
    # The captured iteration (with the whole V-cycle inside) is cached on the
    # projector per (preconditioner, lambda) together with its static buffers,
    # so repeated solves replay it instead of re-capturing (no x_ex tracking:
    # the error terms read a per-solve buffer).
    owner = precond if precond is not None else w
    # unsharded, vectors of <= 2^20 elements: the reductions' last
    # level, the scalar recurrences and the vector updates run fused
    # (wmg_cgls_update / wmg_cgls_direction: same arithmetic, 5 launches fewer)
    fused = (FUSED_CGLS and not getattr(w, "collectives", False)
             and max(M_, Nn) <= (1 << 20))
    key = (id(w), lam, str(dev), fused)
    cache = None if errs.active else owner.__dict__.setdefault("_cgls_graph_cache", {})
    ctx = cache.get(key) if cache is not None else None
    if ctx is not None and ctx["wref"]() is not w:
        ctx = None
    if ctx is None:
        ctx = {"r": t.empty(M_, dtype=t.float64, device=dev),
               "q": t.empty(M_, dtype=t.float64, device=dev),
               "s": t.empty(Nn, dtype=t.float64, device=dev),
               "s_old": t.empty(Nn, dtype=t.float64, device=dev),
               "p": t.empty(Nn, dtype=t.float64, device=dev),
               "x": t.empty(Nn, dtype=t.float64, device=dev),
               "S": t.zeros(16, dtype=t.float64, device=dev),
               "S_host": t.zeros(16, dtype=t.float64).pin_memory(),
               "z": t.empty(Nn, dtype=t.float64, device=dev),
               "loop": None, "loopB": None, "wref": weakref.ref(w)}
        if cache is not None:
            cache[key] = ctx
    r, q, s, s_old, S, S_host = (ctx[k] for k in ("r", "q", "s", "s_old", "S", "S_host"))
    # every solve starts from clean scalars: S[8] is the sticky breakdown flag
    # wmg_cgls_scalars sets, and a cached context must not carry it over
    S.zero_()
    # A preconditioner that already holds its own captured graph (captured at
    # construction, i.e. in the setup) is replayed between two captured halves
    # of the iteration instead of being re-captured inside it.
    split = precond is not None and getattr(precond, "_graph", None) is not None
    ctx["x"].copy_(x)
    x = ctx["x"]
    st = D.stream_handle
    w.forward_(x, q)
    D.axpy(r, bd, 1.0, -1, q)
    w.backward_(r, s)
    if lam != 0:
        D.add_scaled(s, s, lam, -1, x)
    if precond is None:
        z = s
        D.det_reduce([(N.RED_SQ, s, None, None)], out=S[0:1])
        D.det_reduce([(N.RED_SQ, s, None, None)], out=S[5:6])
    else:
        if split:
            z = ctx["z"]
            precond.apply_(s, z)
        else:
            z = precond._eager(s)
        D.det_reduce([(N.RED_SQ, s, None, None), (N.RED_DOT, z, s, None)], out=S[5:7])
        S[0:1].copy_(S[6:7])
    p = ctx["p"]
    p.copy_(z)
    S[11:12].copy_(S[0:1])                # gamma's second slot (fused kernels)
    if errs.active:
        S[9:11].copy_(errs.device_terms(x))
    S_host.copy_(S, non_blocking=True)
    t.cuda.current_stream(dev).synchronize()
    h = S_host.numpy()
    s0 = float(np.sqrt(h[5]))
    e2, einf = errs.finish(h[9:11]) if errs.active else (None, None)
    record.log(0, 1.0, e2, einf, time.perf_counter() - t0)
    if s0 == 0.0:
        record.status = STATUS_CONVERGED
        return D.to_caller(x.clone(), was_np), record

    n_img, n_sino = Nn, M_
    # weak references: the cache lives on the preconditioner (or projector), so
    # the captured body must not keep either alive
    wref = weakref.ref(w)
    pref = weakref.ref(precond) if precond is not None else None

    def body():
        w = wref()
        precond = pref() if pref is not None else None
        w.forward_(p, q)
        if fused:
            part = D.det_partials([(N.RED_SQ, q, None, None)])
            # (the two reductions have different lengths: separate chunk sums)
            part_pp = D.det_partials([(N.RED_SQ, p, None, None)], slot=1) if lam != 0 else None
            N.call("wmg_cgls_update", n_img, n_sino, D.ptr(x), D.ptr(p), D.ptr(r), D.ptr(q),
                   D.ptr(part), D.ptr(part_pp), float(lam), D.ptr(S), st())
        else:
            D.det_reduce([(N.RED_SQ, q, None, None)], out=S[1:2])
            _sino(w, S[1:2])              # angle shards: sum of the ranks' partials
            if lam != 0:
                D.det_reduce([(N.RED_SQ, p, None, None)], out=S[2:3])
            N.call("wmg_cgls_scalars", D.ptr(S), float(lam), 0, st())
            N.call("wmg_axpy_dev", n_img, D.ptr(x), D.ptr(x), D.ptr(S[3:4]), 1, D.ptr(p), st())
            N.call("wmg_axpy_dev", n_sino, D.ptr(r), D.ptr(r), D.ptr(S[3:4]), -1, D.ptr(q),
                   st())
        if precond is not None:
            s_old.copy_(s)
        w.backward_(r, s)
        if lam != 0:
            D.add_scaled(s, s, lam, -1, x)
        if precond is None:
            if fused:
                part = D.det_partials([(N.RED_SQ, s, None, None)])
                N.call("wmg_cgls_direction", n_img, D.ptr(p), D.ptr(s), D.ptr(part), 1,
                       D.ptr(S), st())
            else:
                D.det_reduce([(N.RED_SQ, s, None, None)], out=S[5:6])
                N.call("wmg_cgls_scalars", D.ptr(S), float(lam), 1, st())
                N.call("wmg_lincomb_dev", n_img, D.ptr(p), 1.0, D.ptr(s), D.ptr(S[4:5]),
                       D.ptr(p), st())
            tail()
        elif not split:
            tail(precond._eager(s))

    def tail(zz=None):
        if zz is not None and fused:
            part = D.det_partials([(N.RED_SQ, s, None, None), (N.RED_DOT, zz, s, None),
                                   (N.RED_DOTDIFF, zz, s, s_old)])
            N.call("wmg_cgls_direction", n_img, D.ptr(p), D.ptr(zz), D.ptr(part), 2,
                   D.ptr(S), st())
        elif zz is not None:
            D.det_reduce([(N.RED_SQ, s, None, None), (N.RED_DOT, zz, s, None),
                          (N.RED_DOTDIFF, zz, s, s_old)], out=S[5:8])
            N.call("wmg_cgls_scalars", D.ptr(S), float(lam), 2, st())
            N.call("wmg_lincomb_dev", n_img, D.ptr(p), 1.0, D.ptr(zz), D.ptr(S[4:5]),
                   D.ptr(p), st())
        if errs.active:
            S[9:11].copy_(errs.device_terms(x))
        S_host.copy_(S, non_blocking=True)

    zbuf = ctx["z"]
    loop = ctx["loop"]
    if loop is None:
        loop = ctx["loop"] = _GraphedLoop(body, bool(getattr(w, "collectives", False)))
    loop_b = ctx["loopB"]
    if split and loop_b is None:
        loop_b = ctx["loopB"] = _GraphedLoop(lambda: tail(zbuf),
                                             bool(getattr(w, "collectives", False)))
    for k in range(1, cfg.max_iterations + 1):
        loop.step()
        if split:
            precond.apply_(s, zbuf)          # the preconditioner's own graph
            loop_b.step()
        t.cuda.current_stream(dev).synchronize()
        h = S_host.numpy()
        if h[8] != 0.0:
            record.status = STATUS_BREAKDOWN
            break
        rel = float(np.sqrt(h[5])) / s0
        e2, einf = errs.finish(h[9:11]) if errs.active else (None, None)
        record.log(k, rel, e2, einf, time.perf_counter() - t0)
        if cfg.residual_tolerance > 0 and rel < cfg.residual_tolerance:
            record.status = STATUS_CONVERGED
            break
        if h[11 if fused else 0] == 0.0:      # gamma
            record.status = STATUS_CONVERGED
            break
    else:
        record.status = STATUS_MAX_ITERATIONS
    return D.to_caller(x.clone(), was_np), record


# --------------------------------------------------------------- CGLS family
def cgls_solve(w, b, precond=None, x0=None, cfg: SolverConfig = None, x_ex=None,
               graph: bool = True):
    """CGLS on min ||W x - b||^2 + lam ||x||^2; with ``precond`` (an operator
    approximating (W^T W + lam I)^-1, e.g. ``wmg_preconditioner``) the flexible
    Polak-Ribiere PCG on the normal equations ("WMG-CGLS").

      r = b - W x;  s = W^T r - lam x;  z = M s;  p = z;  gamma = <z, s>
      loop: q = W p;  delta = <q,q> + lam <p,p>;  alpha = gamma / delta
            x += alpha p;  r -= alpha q;  s_new = W^T r - lam x
            z = M s_new;  beta = <z, s_new - s> / gamma   (M = I: <s,s>/gamma)
            gamma = <z, s_new>;  p = z + beta p
    Logged residual: ||s_k|| / ||s_0|| (normal-equations recurrence residual).

    With ``graph=True`` (default, when W and the preconditioner are our device
    operators) the scalars stay on the device and each iteration is one CUDA
    graph replay; results are bit-identical to the eager path.
    """
    t = D.require_cuda()
    if cfg is None:
        cfg = SolverConfig()
    M_, Nn = w.shape
    bd, was_np = D.to_device(b)
    if bd.numel() != M_:
        raise DimensionMismatchError("cgls_solve: b length mismatch")
    if x0 is None:
        x = t.zeros(Nn, dtype=t.float64, device=bd.device)
    else:
        x = D.to_device(x0)[0].clone()
        if x.numel() != Nn:
            raise DimensionMismatchError("cgls_solve: x0 length mismatch")
    lam = float(cfg.regularization_lambda)
    errs = _ErrorTracker(x_ex, Nn, bd.device)
    record = ConvergenceRecord()
    t0 = time.perf_counter()
    if graph and _graphable(w, precond):
        return _cgls_graphed(w, bd, x, lam, precond, cfg, errs, was_np, record, t0)
    minv = _as_device_op(precond)

    dev = bd.device
    r = t.empty(M_, dtype=t.float64, device=dev)
    q = t.empty(M_, dtype=t.float64, device=dev)
    s = t.empty(Nn, dtype=t.float64, device=dev)
    s_old = t.empty(Nn, dtype=t.float64, device=dev)
    w.forward_(x, q)
    D.axpy(r, bd, 1.0, -1, q)                         # r = b - W x
    w.backward_(r, s)                                 # s = W^T r
    if lam != 0:
        D.add_scaled(s, s, lam, -1, x)                # s -= lam x
    z = s if minv is None else minv(s)
    p = z.clone()
    if minv is None:
        h = _readback(D.det_norm_sq(s), errs.device_terms(x))
        gamma = float(h[0])
        s0 = float(np.sqrt(gamma))
        eterms = h[1:3]
    else:
        h = _readback(D.det_reduce([(N.RED_SQ, s, None, None), (N.RED_DOT, z, s, None)]),
                      errs.device_terms(x))
        s0 = float(np.sqrt(h[0]))
        gamma = float(h[1])
        eterms = h[2:4]
    e2, einf = errs.finish(eterms) if errs.active else (None, None)
    record.log(0, 1.0, e2, einf, time.perf_counter() - t0)
    if s0 == 0.0:
        record.status = STATUS_CONVERGED
        return D.to_caller(x, was_np), record

    for k in range(1, cfg.max_iterations + 1):
        w.forward_(p, q)
        if lam != 0:
            hd = _readback(_sino(w, D.det_norm_sq(q)), D.det_norm_sq(p))
            delta = float(hd[0]) + lam * float(hd[1])
        else:
            delta = float(_readback(_sino(w, D.det_norm_sq(q)))[0])
        if delta <= 0.0 or not np.isfinite(delta):
            record.status = STATUS_BREAKDOWN
            return D.to_caller(x, was_np), record
        alpha = gamma / delta
        D.axpy(x, x, alpha, +1, p)
        D.axpy(r, r, alpha, -1, q)
        if minv is not None:
            s_old.copy_(s)
        w.backward_(r, s)
        if lam != 0:
            D.add_scaled(s, s, lam, -1, x)
        if minv is None:
            h = _readback(D.det_norm_sq(s), errs.device_terms(x))
            gnew = float(h[0])
            snorm = float(np.sqrt(gnew))
            eterms = h[1:3]
        else:
            z = minv(s)
            h = _readback(D.det_reduce([(N.RED_SQ, s, None, None), (N.RED_DOT, z, s, None),
                                        (N.RED_DOTDIFF, z, s, s_old)]),
                          errs.device_terms(x))
            snorm = float(np.sqrt(h[0]))
            gnew = float(h[1])
            pr = float(h[2])
            eterms = h[3:5]
        rel = snorm / s0
        e2, einf = errs.finish(eterms) if errs.active else (None, None)
        record.log(k, rel, e2, einf, time.perf_counter() - t0)
        if cfg.residual_tolerance > 0 and rel < cfg.residual_tolerance:
            record.status = STATUS_CONVERGED
            return D.to_caller(x, was_np), record
        if minv is None:
            beta = gnew / gamma
            gamma = gnew
            D.lincomb(p, 1.0, s, beta, p)             # p = s + beta p
        else:
            beta = pr / gamma
            gamma = gnew
            D.lincomb(p, 1.0, z, beta, p)             # p = z + beta p
        if gamma == 0.0:
            record.status = STATUS_CONVERGED
            return D.to_caller(x, was_np), record
    record.status = STATUS_MAX_ITERATIONS
    return D.to_caller(x, was_np), record


# -------------------------------------------------------------------- GMRES
def gmres_solve(op, f, precond=None, x0=None, cfg: SolverConfig = None, x_ex=None,
                restart: int = 100):
    """Right-preconditioned restarted GMRES on op x = f (op = normal operator).

    Arnoldi with classical Gram-Schmidt applied twice (CGS2): the projections
    stay on the device (DET_SUM, 8 per launch) and each Arnoldi step reads back
    its Hessenberg column and ||w|| once; Givens rotations on the host
    (O(restart^2) scalars).  Logged residual: the GMRES residual
    estimate |g_{j+1}| / ||f - op x0||, i.e. the normal-equations residual.
    """
    t = D.require_cuda()
    if cfg is None:
        cfg = SolverConfig()
    if restart < 1:
        raise ValueError("restart must be >= 1")
    fd, was_np = D.to_device(f)
    n = fd.numel()
    x = t.zeros_like(fd) if x0 is None else D.to_device(x0)[0].clone()
    if x.shape != fd.shape:
        raise DimensionMismatchError("gmres_solve: x0/f length mismatch")
    A = _as_device_op(op)
    minv = (lambda v: v) if precond is None else _as_device_op(precond)
    errs = _ErrorTracker(x_ex, n, fd.device)
    record = ConvergenceRecord()
    t0 = time.perf_counter()
    dev = fd.device
    m = int(restart)
    V = t.empty((m + 1, n), dtype=t.float64, device=dev)
    Z = t.empty((m, n), dtype=t.float64, device=dev) if precond is not None else None
    r = t.empty_like(fd)
    D.axpy(r, fd, 1.0, -1, A(x))
    h0 = _readback(D.det_norm_sq(r), errs.device_terms(x))
    beta0 = float(np.sqrt(h0[0]))
    res_norm0 = beta0
    e2, einf = errs.finish(h0[1:3]) if errs.active else (None, None)
    record.log(0, 1.0, e2, einf, time.perf_counter() - t0)
    if res_norm0 == 0.0:
        record.status = STATUS_CONVERGED
        return D.to_caller(x, was_np), record
    k = 0
    beta = beta0
    hbuf = t.empty(m + 1, dtype=t.float64, device=dev)
    hacc = t.zeros(m + 2, dtype=t.float64, device=dev)
    while True:
        D.scale(V[0], 1.0 / beta, r)
        H = np.zeros((m + 1, m))
        cs = np.zeros(m)
        sn = np.zeros(m)
        g = np.zeros(m + 1)
        g[0] = beta
        j_done = 0
        stop = None
        for j in range(m):
            k += 1
            zj = minv(V[j])
            if Z is not None:
                Z[j].copy_(zj)
            wv = A(zj)
            wv = wv.clone() if wv.data_ptr() == zj.data_ptr() else wv
            # CGS2 with the projections kept on the device: both passes, their
            # sum (the oracle's hcol += hh, same order) and ||w||^2 come back to
            # the host in ONE read per Arnoldi step
            hacc.zero_()
            for _ in range(2):
                specs = [(N.RED_DOT, V[i], wv, None) for i in range(j + 1)]
                for c0 in range(0, len(specs), 8):
                    D.det_reduce(specs[c0:c0 + 8], out=hbuf[c0:min(c0 + 8, j + 1)])
                N.call("wmg_cgs_update", n, j + 1, D.ptr(wv), D.ptr(V), n, D.ptr(hbuf),
                       D.stream_handle())
                hacc[: j + 1].add_(hbuf[: j + 1])
            D.det_reduce([(N.RED_SQ, wv, None, None)], out=hacc[m + 1:m + 2])
            hv = _readback(hacc[: j + 1], hacc[m + 1:m + 2])
            hcol = np.zeros(j + 2)
            hcol[: j + 1] = hv[: j + 1]
            hn = float(np.sqrt(hv[j + 1]))
            hcol[j + 1] = hn
            # apply previous rotations
            for i in range(j):
                a_, b_ = hcol[i], hcol[i + 1]
                hcol[i] = cs[i] * a_ + sn[i] * b_
                hcol[i + 1] = -sn[i] * a_ + cs[i] * b_
            den = np.hypot(hcol[j], hcol[j + 1])
            cs[j] = hcol[j] / den if den else 1.0
            sn[j] = hcol[j + 1] / den if den else 0.0
            hcol[j] = den
            hcol[j + 1] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            H[: j + 2, j] = hcol
            j_done = j + 1
            rel = abs(g[j + 1]) / res_norm0
            happy = hn == 0.0
            if not happy:
                D.scale(V[j + 1], 1.0 / hn, wv)
            last = (k >= cfg.max_iterations or happy or
                    (cfg.residual_tolerance > 0 and rel < cfg.residual_tolerance))
            if errs.active or last or j == m - 1:
                # materialise x_k = x + Z y for logging / exit
                y = np.linalg.solve(np.triu(H[:j_done, :j_done]), g[:j_done]) if j_done else []
                xk = _gmres_update(x, V, Z, y, precond, minv, n)
                if errs.active:
                    e2, einf = errs.finish(_readback(errs.device_terms(xk)))
                else:
                    e2 = einf = None
                record.log(k, rel, e2, einf, time.perf_counter() - t0)
                if last or j == m - 1:
                    x = xk
                    if happy or (cfg.residual_tolerance > 0 and rel < cfg.residual_tolerance):
                        stop = STATUS_CONVERGED
                    elif k >= cfg.max_iterations:
                        stop = STATUS_MAX_ITERATIONS
                    break
            else:
                record.log(k, rel, None, None, time.perf_counter() - t0)
        if stop is not None:
            record.status = stop
            return D.to_caller(x, was_np), record
        # restart
        D.axpy(r, fd, 1.0, -1, A(x))
        beta = float(np.sqrt(_readback(D.det_norm_sq(r))[0]))
        if beta == 0.0:
            record.status = STATUS_CONVERGED
            return D.to_caller(x, was_np), record


def _gmres_update(x, V, Z, y, precond, minv, n):
    t = D.torch()
    k = len(y)
    xk = x.clone()
    if k == 0:
        return xk
    cf = t.as_tensor(np.asarray(y, dtype=np.float64), device=x.device)
    if precond is None:
        N.call("wmg_combo", n, k, D.ptr(xk), D.ptr(V), n, D.ptr(cf), 1, D.stream_handle())
    else:
        N.call("wmg_combo", n, k, D.ptr(xk), D.ptr(Z), n, D.ptr(cf), 1, D.stream_handle())
    return xk
