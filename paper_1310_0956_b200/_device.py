"""Device-buffer plumbing shared by the operator and solver layers.

PyTorch supplies HBM buffers and the current CUDA stream; every arithmetic op on
the hot path is one of our sm_100a kernels called through the C ABI
(``_native``).  Vectors arrive as numpy arrays (copied to HBM, results copied
back -- the reference's calling convention) or as torch CUDA tensors (kept
resident).
"""
from __future__ import annotations

import ctypes
import threading
import weakref

import numpy as np

from . import _native as N

_scratch = {}


def torch():
    import torch as _t
    return _t


def require_cuda():
    t = torch()
    N.load(require_gpu=True)
    return t


def stream_handle():
    t = torch()
    return ctypes.c_void_p(t.cuda.current_stream().cuda_stream)


def ptr(tensor):
    return ctypes.c_void_p(tensor.data_ptr()) if tensor is not None else None


def is_torch(v) -> bool:
    try:
        import torch as _t
    except ImportError:  # pragma: no cover
        return False
    return isinstance(v, _t.Tensor)


def to_device(v, dtype=None, device=None):
    """Return (tensor on GPU, was_numpy)."""
    t = require_cuda()
    dtype = dtype or t.float64
    if is_torch(v):
        if v.is_cuda:
            out = v
            if out.dtype != dtype:
                out = out.to(dtype)
            return out.contiguous(), False
        return v.to(device=device or "cuda", dtype=dtype).contiguous(), True
    a = np.ascontiguousarray(np.asarray(v), dtype=np.float64 if dtype == t.float64 else np.float32)
    dev = t.device(device) if device is not None else t.device("cuda", t.cuda.current_device())
    if a.nbytes >= _STAGE_MIN_BYTES:
        h = t.from_numpy(a)
        if h.is_pinned():
            # already page-locked (e.g. a previous result handed out from the
            # pinned pool, as in the reference's ``w.T @ (w @ v)``): one DMA
            out = t.empty(a.size, dtype=dtype, device=dev)
            out.copy_(h, non_blocking=True)
            t.cuda.current_stream(dev).synchronize()   # the caller may reuse the array
            return out, True
        return _h2d_staged(a, dtype, dev), True
    return t.from_numpy(a).to(dev, non_blocking=False), True


# Host <-> device copies of large numpy vectors (the reference-style call
# ``w @ x`` with numpy in and out).  Measured on the B200 box (64-95 MB):
# pageable H2D 10.9 GB/s, ``.cpu()`` D2H 2.1 GB/s; pinned copies 47-57 GB/s.
# H2D: ``wmg_h2d_staged`` (csrc/hostio.cu) copies the array into a cached
# pinned staging buffer with a pool of native host threads (no GIL) in 4 MB
# chunks and issues each chunk's DMA as soon as it has landed.  D2H: into a
# pinned buffer from a small pool, returned as the numpy view itself.
_STAGE_MIN_BYTES = 64 << 10         # below: plain pageable copies (latency bound anyway)
_STAGE_THREADS = 6                   # host-copy threads (tools/probe_h2d_threads.py: 4-6 saturate
                                     # the box's ~25 GB/s pageable -> pinned copy rate; more are slower)
_stage = {}
_stage_lock = threading.Lock()


def _h2d_staged(a, dtype, dev):
    from . import _native as N
    t = torch()
    key = (str(dev), threading.get_ident())
    with _stage_lock:
        ent = _stage.get(key)
    if ent is None or ent[0].numel() < a.nbytes:
        buf = t.empty(max(a.nbytes, 1), dtype=t.uint8).pin_memory()
        ent = (buf, t.cuda.Event())
        with _stage_lock:
            _stage[key] = ent
    buf, done = ent
    done.synchronize()                       # the previous DMA out of this buffer
    out = t.empty(a.size, dtype=dtype, device=dev)
    stream = t.cuda.current_stream(dev)
    N.call("wmg_h2d_staged", out.data_ptr(), a.ctypes.data, a.nbytes, buf.data_ptr(),
           _STAGE_THREADS, stream.cuda_stream)
    done.record(stream)
    return out


# Results returned to numpy callers live in pinned buffers from a small pool per
# (shape, dtype): a buffer is reused once the numpy array handed out for it (and
# every array derived from it, which keeps it alive) is gone -- tracked with a
# weak reference -- so a caller that keeps the last few results still gets
# 56 GB/s DMA without a cudaHostAlloc per call; past _D2H_POOL live results,
# results go to pageable memory (16 GB/s).
_D2H_POOL = 4
_d2h = {}


def _IN_USE():
    return True


def _d2h_buffer(shape, dtype):
    t = torch()
    key = (tuple(shape), dtype)
    with _stage_lock:
        pool = _d2h.setdefault(key, [])
        for ent in pool:
            if ent[1] is None or ent[1]() is None:
                ent[1] = _IN_USE               # reserved until the caller's array exists
                return ent
        if len(pool) < _D2H_POOL:
            ent = [t.empty(shape, dtype=dtype, pin_memory=True), _IN_USE]
            pool.append(ent)
            return ent
    return None


def to_caller(tensor, was_numpy):
    if was_numpy:
        tt = tensor.detach()
        if tt.is_cuda and tt.numel() * tt.element_size() >= _STAGE_MIN_BYTES:
            t = torch()
            ent = _d2h_buffer(tt.shape, tt.dtype)
            if ent is None:                    # many live results: pageable copy
                out = np.empty(tuple(tt.shape), dtype=t.empty(0, dtype=tt.dtype).numpy().dtype)
                t.from_numpy(out).copy_(tt)
                return out
            ent[0].copy_(tt, non_blocking=True)
            t.cuda.current_stream(tt.device).synchronize()
            arr = ent[0].numpy()
            ent[1] = weakref.ref(arr)
            return arr
        return tt.cpu().numpy()
    return tensor


_gc_lock = threading.Lock()
_gc_depth = 0
_gc_was_enabled = False


def _gc_pause():
    """Disable the cyclic GC while any thread captures (reference-counted:
    concurrent captures from several host threads nest)."""
    import gc
    global _gc_depth, _gc_was_enabled
    with _gc_lock:
        if _gc_depth == 0:
            _gc_was_enabled = gc.isenabled()
            gc.disable()
        _gc_depth += 1


def _gc_resume():
    import gc
    global _gc_depth
    with _gc_lock:
        _gc_depth -= 1
        if _gc_depth == 0 and _gc_was_enabled:
            gc.enable()


def capture_graph(fn, device):
    """Capture fn() into a new CUDA graph on a side stream (private memory pool)
    and return (graph, fn's result).  Unlike ``torch.cuda.graph`` this does not
    empty the caching allocator first: a capture right after a hierarchy build
    would otherwise pay ~10 ms of cudaFree for the released setup buffers."""
    t = torch()
    cur = t.cuda.current_stream(device)
    side = t.cuda.Stream(device=device)
    side.wait_stream(cur)
    g = t.cuda.CUDAGraph()
    # no cyclic garbage collection while capturing: collecting an unreachable
    # earlier preconditioner would destroy its CUDA graph mid-capture, which
    # invalidates the capture
    _gc_pause()
    try:
        with t.cuda.stream(side):
            # thread-local capture: solves running concurrently in other host
            # threads (their own streams) may keep launching while this one captures
            g.capture_begin(capture_error_mode="thread_local")
            try:
                out = fn()
            finally:
                g.capture_end()
    finally:
        _gc_resume()
    cur.wait_stream(side)
    return g, out


def scratch(n: int, K: int, device, slot: int = 0):
    """Cached device scratch for wmg_det_reduce (+ K result slots), per stream.
    Inside a graph capture a fresh buffer comes from the graph's private pool,
    so two captured graphs never share scratch (they may replay concurrently)."""
    t = torch()
    L = N.load()
    need = int(L.wmg_det_scratch_len(int(n), int(K))) + 16
    if t.cuda.is_current_stream_capturing():
        return t.empty(max(need, 4096), dtype=t.float64, device=device)
    key = (str(device), t.cuda.current_stream(device).cuda_stream, slot)
    buf = _scratch.get(key)
    if buf is None or buf.numel() < need:
        buf = t.empty(max(need, 4096), dtype=t.float64, device=device)
        _scratch[key] = buf
    return buf


def det_reduce(specs, n=None, out=None):
    """Deterministic float64 reductions (DET_SUM, see csrc/vecops.cu).

    ``specs`` is a list of (op, a, b, c) tuples of CUDA float64 tensors of equal
    length.  Returns a float64 CUDA tensor with one result per spec (no sync).
    """
    t = torch()
    K = len(specs)
    if not 1 <= K <= 8:
        raise ValueError("det_reduce takes 1..8 reductions")
    a0 = specs[0][1]
    n = a0.numel() if n is None else n
    for sp_ in specs:
        for v in sp_[1:]:
            if v is not None and v.numel() != n:
                raise ValueError("det_reduce operands must have equal lengths")
    dev = a0.device
    sc = scratch(n, K, dev)
    if out is None:
        out = t.empty(K, dtype=t.float64, device=dev)
    ops = (ctypes.c_int * K)(*[int(s[0]) for s in specs])
    A = (ctypes.c_void_p * K)(*[s[1].data_ptr() for s in specs])
    B = (ctypes.c_void_p * K)(*[(s[2].data_ptr() if s[2] is not None else 0) for s in specs])
    C = (ctypes.c_void_p * K)(*[(s[3].data_ptr() if len(s) > 3 and s[3] is not None else 0)
                                for s in specs])
    N.call("wmg_det_reduce", int(n), K, ops, A, B, C, ptr(sc), ptr(out), stream_handle())
    return out


def det_partials(specs, slot=0):
    """Level 1 of ``det_reduce`` only: returns the scratch tensor holding the
    chunk sums (reduction k at offset k * ceil(n / 1024)), for the fused CGLS
    kernels that finish the reduction themselves.  ``slot``: which of the
    stream's scratch buffers to use (two sets of chunk sums alive at once)."""
    K = len(specs)
    a0 = specs[0][1]
    n = a0.numel()
    for sp_ in specs:
        for v in sp_[1:]:
            if v is not None and v.numel() != n:
                raise ValueError("det_partials operands must have equal lengths")
    sc = scratch(n, K, a0.device, slot)
    ops = (ctypes.c_int * K)(*[int(s[0]) for s in specs])
    A = (ctypes.c_void_p * K)(*[s[1].data_ptr() for s in specs])
    B = (ctypes.c_void_p * K)(*[(s[2].data_ptr() if s[2] is not None else 0) for s in specs])
    C = (ctypes.c_void_p * K)(*[(s[3].data_ptr() if len(s) > 3 and s[3] is not None else 0)
                                for s in specs])
    N.call("wmg_det_partials", int(n), K, ops, A, B, C, ptr(sc), stream_handle())
    return sc


def det_dot(a, b):
    return det_reduce([(N.RED_DOT, a, b, None)])


def det_norm_sq(a):
    return det_reduce([(N.RED_SQ, a, None, None)])


def maxabs(a, b=None):
    t = torch()
    out = t.empty(1, dtype=t.float64, device=a.device)
    N.call("wmg_maxabs", a.numel(), ptr(a), ptr(b), ptr(out), stream_handle())
    return out


def axpy(out, y, alpha, sgn, x):
    N.call("wmg_axpy", out.numel(), ptr(out), ptr(y), float(alpha), int(sgn), ptr(x),
           stream_handle())
    return out


def lincomb(out, a, x, b, y, c=0.0, z=None):
    N.call("wmg_lincomb", out.numel(), ptr(out), float(a), ptr(x), float(b), ptr(y), float(c),
           ptr(z), stream_handle())
    return out


def add_scaled(out, g, lam, sgn, v):
    N.call("wmg_add_scaled", out.numel(), ptr(out), ptr(g), float(lam), int(sgn), ptr(v),
           stream_handle())
    return out


def smooth_update(z, omega, c, r, az=None):
    """z += omega * (c .* (r - az)) in one kernel (az None: az = 0)."""
    N.call("wmg_smooth_update", z.numel(), ptr(z), float(omega), ptr(c), ptr(r), ptr(az),
           stream_handle())
    return z


def smooth_update_batch(Z, omegas, scalings, R, AZ=None):
    """Z[b] += omegas[b] * (scalings[b] .* (R[b] - AZ[b])) for a batch of node
    smoothers in one launch (rows of Z, R, AZ contiguous; bit-identical to
    ``smooth_update`` per row)."""
    B = Z.shape[0]
    om = (ctypes.c_double * B)(*[float(o) for o in omegas])
    cs = (ctypes.c_void_p * B)(*[c.data_ptr() for c in scalings])
    N.call("wmg_smooth_update_batch", int(Z.shape[1]), B, ptr(Z), om, cs, ptr(R),
           ptr(AZ) if AZ is not None else None, stream_handle())
    return Z


def hadamard(out, x, y):
    N.call("wmg_scale", out.numel(), ptr(out), 1.0, ptr(x), ptr(y), stream_handle())
    return out


def scale(out, a, x):
    N.call("wmg_scale", out.numel(), ptr(out), float(a), ptr(x), None, stream_handle())
    return out


def recip(out, s):
    N.call("wmg_recip", out.numel(), ptr(out), ptr(s), stream_handle())
    return out


def error_metrics_dev(x, x_ex, ex_norm2=None, ex_inf=None):
    """Device-side rel-L2 / rel-Linf (phantom.py:64-75); returns a CUDA tensor
    [sum (x-x_ex)^2, max|x-x_ex|] plus the precomputed exact-image norms."""
    t = torch()
    r = det_reduce([(N.RED_SQDIFF, x, x_ex, None)])
    m = maxabs(x, x_ex)
    return t.cat([r, m])
