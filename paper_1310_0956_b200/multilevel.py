"""Haar intergrid operators, the WMG hierarchy and the WTG V-cycle on B200.

Drop-in for /root/reference/pkg/src/wmgtomo/multilevel.py:
  * ``BAND_IDS``, ``haar_scaling_1d``, ``haar_wavelet_1d``, ``IntergridSet``,
    ``build_intergrid_set`` (:28-79) -- host descriptors (scipy CSR, small),
    identical to the reference; the device applies them with the
    ``wmg_haar_restrict`` / ``wmg_haar_prolong`` kernels (same coefficients
    +-0.4999999999999999 and summation order);
  * ``WmgNode`` / ``WmgHierarchy`` / ``build_wmg_hierarchy`` (:82-166): the
    internal-node systems P^T P + lam I with P = W R_path^T are applied
    MATRIX-FREE (prolong along the path -> projector pair -> restrict); only
    the coarsest (leaf) Grams are assembled -- directly from the exact ray walk
    (wmg_leaf_factor) and a float64 GEMM -- and Cholesky-factored in HBM;
  * ``wtg_apply`` (:175-198, hybrid and multiplicative), ``wmg_preconditioner``
    (:201-208).

Extension (BASELINE configs 1/2/4: "2 pre- and 2 post-smoothing SIRT sweeps per
level"; not defined by the reference, SURVEY.md s8 a16 option (ii)): with
``nu_pre``/``nu_post`` > 0 every internal node applies
    z <- z + omega_p C_p (v - A_p z),
    C_p = 1 / (2^-k * sum of W's column sums over each coarse pixel block),
    omega_p = 0.95 / lambda_max(C_p A_p)   (10 power iterations at setup)
before and after its wavelet two-grid correction.  nu_pre = nu_post = 0 (the
default) is exactly the reference's smoother-free cycle.
``classical_tg_preconditioner`` is provided as well.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np
import scipy.sparse as sp

from . import _device as D
from . import _native as N
from .sparse_kernels import (DenseFactorization, DimensionMismatchError,
                             NotPositiveDefiniteError, spd_inverse_)

BAND_IDS = ("LL", "LH", "HL", "HH")
BAND_CODE = {"LL": 0, "LH": 1, "HL": 2, "HH": 3}


def _check_even(n: int):
    if n < 2 or n % 2 != 0:
        raise ValueError(f"grid side must be even and >= 2, got {n}")


def haar_scaling_1d(n: int) -> sp.csr_matrix:
    """(n/2)-by-n averaging operator: row k = 1/sqrt(2) at columns 2k, 2k+1."""
    _check_even(n)
    h = n // 2
    return sp.csr_matrix((np.full(n, 1.0 / np.sqrt(2.0)), (np.repeat(np.arange(h), 2),
                                                           np.arange(n))), shape=(h, n))


def haar_wavelet_1d(n: int) -> sp.csr_matrix:
    """(n/2)-by-n differencing operator: row k = (1, -1)/sqrt(2) at 2k, 2k+1."""
    _check_even(n)
    h = n // 2
    vals = np.tile([1.0, -1.0], h) / np.sqrt(2.0)
    return sp.csr_matrix((vals, (np.repeat(np.arange(h), 2), np.arange(n))), shape=(h, n))


@dataclass(frozen=True)
class IntergridSet:
    """The four orthonormal restrictions for one coarsening step of an n-grid."""

    n: int
    restrictions: dict

    def __getitem__(self, band: str) -> sp.csr_matrix:
        return self.restrictions[band]


def build_intergrid_set(n: int) -> IntergridSet:
    """kron(row factor, col factor); the row factor acts along y (rows)."""
    _check_even(n)
    s = haar_scaling_1d(n)
    j = haar_wavelet_1d(n)
    return IntergridSet(n=n, restrictions={
        "LL": sp.kron(s, s, format="csr"),
        "LH": sp.kron(j, s, format="csr"),
        "HL": sp.kron(s, j, format="csr"),
        "HH": sp.kron(j, j, format="csr"),
    })


# ------------------------------------------------------------ device kernels
def restrict(side: int, fine, bands, out=None):
    """R_band fine for each band in ``bands`` -> tensor (len(bands), (side/2)^2)."""
    t = D.torch()
    mask = 0
    for b in bands:
        mask |= 1 << BAND_CODE[b]
    order = [b for b in BAND_IDS if (mask >> BAND_CODE[b]) & 1]
    if order != list(bands):
        raise ValueError("bands must be given in LL, LH, HL, HH order")
    nc = (side // 2) ** 2
    if out is None:
        out = t.empty((len(bands), nc), dtype=t.float64, device=fine.device)
    N.call("wmg_haar_restrict", side, D.ptr(fine), mask, D.ptr(out), D.stream_handle())
    return out


def prolong(side: int, coarse, band: str, fine, accumulate: bool):
    """fine = (fine if accumulate else 0) + R_band^T coarse."""
    N.call("wmg_haar_prolong", side, D.ptr(coarse), BAND_CODE[band], D.ptr(fine),
           int(bool(accumulate)), D.stream_handle())
    return fine


def restrict_batch(side: int, fine, bands, out):
    """out[b] = R_band fine[b] for each band, a batch of contiguous items in one
    launch (bit-identical to ``restrict`` per item); out: (B, len(bands), nc)."""
    mask = 0
    for b in bands:
        mask |= 1 << BAND_CODE[b]
    if [b for b in BAND_IDS if (mask >> BAND_CODE[b]) & 1] != list(bands):
        raise ValueError("bands must be given in LL, LH, HL, HH order")
    N.call("wmg_haar_restrict_batch", side, fine.shape[0], D.ptr(fine), mask, D.ptr(out),
           D.stream_handle())
    return out


def prolong_batch(side: int, coarse, bands, fine, accumulate: bool):
    """fine[b] (+)= R_{bands[0]}^T coarse[b, 0] + ... in band order, one launch
    for the batch (bit-identical to successive ``prolong`` calls per item);
    coarse: (B, len(bands), (side/2)^2), fine: (B, side^2)."""
    codes = (N.ctypes.c_int * len(bands))(*[BAND_CODE[b] for b in bands])
    N.call("wmg_haar_prolong_batch", side, fine.shape[0], len(bands), codes, D.ptr(coarse),
           D.ptr(fine), int(bool(accumulate)), D.stream_handle())
    return fine


# Node applications prolong / restrict along the whole band path in one launch
# (wmg_haar_prolong_path / wmg_haar_restrict_path, bit-identical to the
# level-by-level kernels); False: level by level (testing).
FUSED_PATHS = True


def _path_codes(paths):
    depth = len(paths[0])
    arr = (N.ctypes.c_int * (len(paths) * depth))(
        *[BAND_CODE[b] for p in paths for b in p])
    return depth, arr


def prolong_path(n: int, paths, coarse, fine):
    """fine[i] (n*n) = R_{paths[i]}^T coarse[i] for a batch of band paths
    (coarse: (B, (n >> depth)^2), fine: (B, n*n), contiguous rows)."""
    depth, arr = _path_codes(paths)
    N.call("wmg_haar_prolong_path", n, depth, len(paths), arr, D.ptr(coarse), D.ptr(fine),
           D.stream_handle())
    return fine


def restrict_path(n: int, paths, fine, coarse):
    """coarse[i] = R_{paths[i]} fine[i] for a batch of band paths."""
    depth, arr = _path_codes(paths)
    N.call("wmg_haar_restrict_path", n, depth, len(paths), arr, D.ptr(fine), D.ptr(coarse),
           D.stream_handle())
    return coarse


# ------------------------------------------------------------------ nodes
@dataclass
class WmgNode:
    """One subproblem; its system is v -> P^T (P v) + lam v with P = W R_path^T."""

    side: int
    level: int
    path: str
    factor: Optional[object]           # the shared projector (matrix-free P)
    lam: float
    intergrid: Optional[IntergridSet] = None
    children: dict = field(default_factory=dict)
    coarse_solve: Optional[DenseFactorization] = None
    bands: tuple = ()
    hierarchy: Optional["WmgHierarchy"] = field(default=None, repr=False)
    smooth_c: Optional[object] = field(default=None, repr=False)
    smooth_omega: float = 0.0

    @property
    def dim(self) -> int:
        return self.side * self.side

    @property
    def is_coarsest(self) -> bool:
        return self.coarse_solve is not None

    def apply_system_(self, v, out):
        """Device: out = P^T (P v) + lam v (matrix-free)."""
        h = self.hierarchy
        w = h.node_projector
        k = len(self.bands)
        t = D.torch()
        # prolong to the fine grid (coarsest factor first, as R_path^T does)
        sino = h.buf(("sino",), w.shape[0])
        if k and FUSED_PATHS and getattr(w, "supports_forward_path", False):
            # prolongation evaluated inside the forward's padding pass
            w.forward_path_(v.view(1, -1), [self.bands], sino.view(1, -1))
        else:
            cur = v
            if k and FUSED_PATHS:
                cur = prolong_path(h.n, [self.bands], v, h.buf(("pf", 0), h.n * h.n))
            else:
                for lv in range(k - 1, -1, -1):
                    side_f = h.n >> lv
                    buf = h.buf(("pf", lv), side_f * side_f)
                    prolong(side_f, cur, self.bands[lv], buf, accumulate=False)
                    cur = buf
            w.forward_(cur, sino)
        img = h.buf(("img",), w.shape[1]) if k else out
        w.backward_(sino, img)
        cur = img
        if k and FUSED_PATHS:
            restrict_path(h.n, [self.bands], img, out)
        else:
            for lv in range(k):
                side_f = h.n >> lv
                dst = out if lv == k - 1 else h.buf(("rs", lv), (side_f // 2) ** 2)
                restrict(side_f, cur, (self.bands[lv],), out=dst.view(1, -1))
                cur = dst
        if self.lam != 0:
            D.add_scaled(out, out, self.lam, +1, v)
        return out

    def apply_system(self, v):
        t = D.torch()
        vd, was_np = D.to_device(v)
        if vd.numel() != self.dim:
            raise DimensionMismatchError(f"apply_system: length {vd.numel()} != {self.dim}")
        out = t.empty(self.dim, dtype=t.float64, device=vd.device)
        self.apply_system_(vd, out)
        return D.to_caller(out, was_np)


@dataclass(frozen=True)
class WmgHierarchy:
    levels: int
    lam: float
    root: WmgNode
    projector: object = field(default=None, repr=False, compare=False)
    n: int = 0
    nu_pre: int = 0
    nu_post: int = 0
    leaf_factors: object = field(default=None, repr=False, compare=False)
    leaf_inverses: object = field(default=None, repr=False, compare=False)
    node_projector: object = field(default=None, repr=False, compare=False)
    _bufs: dict = field(default_factory=dict, repr=False, compare=False)

    def buf(self, key, numel):
        t = D.torch()
        b = self._bufs.get(key)
        if b is None or b.numel() < numel:
            b = t.empty(numel, dtype=t.float64, device=self.projector.device)
            self._bufs[key] = b
        return b[:numel]

    def nodes(self):
        out = []

        def rec(nd):
            out.append(nd)
            for b in BAND_IDS:
                if b in nd.children:
                    rec(nd.children[b])
        rec(self.root)
        return out


def _leaf_paths(levels):
    paths = [()]
    for _ in range(levels - 1):
        paths = [p + (b,) for p in paths for b in BAND_IDS]
    return paths


def _assemble_leaf_grams(w, n, lam, levels, ray_chunk=None, paths=None, method="sparse",
                         full=True):
    """Gram P_L^T P_L + lam I for every leaf (or the given band paths of depth
    levels-1), batched in HBM.

    method "sparse": ``wmg_leaf_gram`` accumulates the lower triangle per ray
    bundle without forming P_L (fp64 slab weights, <= 1e-12 of the exact
    ones); "dense": exact P_L slabs from the parity walker + DGEMM.
    ``full=False`` leaves the sparse Grams lower-triangular (upper zero): all
    the factorisations read only the lower triangle."""
    t = D.torch()
    depth = levels - 1
    side_c = n >> depth
    p = side_c * side_c
    M = w.shape[0]
    paths = _leaf_paths(levels) if paths is None else [tuple(q) for q in paths]
    grams = t.zeros((len(paths), p, p), dtype=t.float64, device=w.device)
    if method == "sparse":
        overflow = t.zeros(1, dtype=t.int32, device=w.device)
        for li, path in enumerate(paths):
            bands = (N.ctypes.c_int * depth)(*[BAND_CODE[b] for b in path])
            g = grams[li]
            N.call("wmg_leaf_gram", w.handle, depth, bands, D.ptr(g), D.ptr(overflow),
                   D.stream_handle())
            if full:
                low = g.tril()
                g.copy_(low)
                g.add_(low.tril(-1).T)
                del low
            if lam != 0:
                g.diagonal().add_(lam)
        if int(overflow.item()):
            raise RuntimeError("wmg_leaf_gram: ray-bundle window overflow")
        return paths, grams
    if method != "dense":
        raise ValueError(f"unknown Gram method '{method}'")
    if ray_chunk is None:
        # keep the factor slab around 1 GB
        ray_chunk = max(256, min(M, (1 << 30) // (8 * p)))
    P = t.empty((min(ray_chunk, M), p), dtype=t.float64, device=w.device)
    for li, path in enumerate(paths):
        bands = (N.ctypes.c_int * depth)(*[BAND_CODE[b] for b in path])
        for r0 in range(0, M, ray_chunk):
            nr = min(ray_chunk, M - r0)
            Pc = P[:nr]
            Pc.zero_()
            N.call("wmg_leaf_factor", w.handle, depth, bands, r0, nr, D.ptr(Pc),
                   D.stream_handle())
            grams[li].addmm_(Pc.T, Pc)
        if lam != 0:
            grams[li].diagonal().add_(lam)
    # (the Cholesky reads the lower triangle only; no symmetrisation copy needed)
    return paths, grams


def _is_sharded(w) -> bool:
    """An AngleShardedProjector (sharding.py) spanning more than one rank."""
    return (hasattr(w, "local") and hasattr(w, "reduce_sino_")
            and getattr(w, "collectives", getattr(w, "world", 1) > 1))


def build_wmg_hierarchy(w, n: int, lam: float, levels: int, nu_pre: int = 0,
                        nu_post: int = 0, node_mode: str = "fast",
                        gram: str = "sparse", packed: bool = True) -> WmgHierarchy:
    """Recursive 4-way splitting of W (multilevel.py:151-166), matrix-free.

    ``node_mode``: projector of the internal node systems -- "fast" (float64
    fast kernels, <= 1e-12 relative, default), "fast32" (float32 arithmetic on
    float64 vectors, <= 1e-5 relative: a cheaper, slightly inexact V-cycle for
    flexible outer solvers) or "parity".  ``gram``: leaf Gram assembly --
    "sparse" (per-ray-bundle accumulation, default) or "dense" (exact parity
    P_L + DGEMM, O(M p^2) per leaf).  ``packed``: keep the leaf inverses as
    packed symmetric tiles (half the bytes per coarse solve) when the leaf
    order is a multiple of 128; else dense row-major.
    """
    if levels < 2:
        raise ValueError("levels must be >= 2")
    if lam < 0:
        raise ValueError("lambda must be nonnegative")
    if n % (2 ** (levels - 1)) != 0:
        raise ValueError(f"n={n} is not divisible by 2^(levels-1)={2 ** (levels - 1)}")
    if nu_pre < 0 or nu_post < 0:
        raise ValueError("smoothing counts must be nonnegative")
    if w.shape[1] != n * n:
        raise DimensionMismatchError(f"projector has {w.shape[1]} columns, expected {n * n}")
    sharded = _is_sharded(w)
    base = w.local if sharded else w
    if not hasattr(base, "handle"):
        raise TypeError("build_wmg_hierarchy needs a LineProjector (build_projector) or an "
                        "AngleShardedProjector")
    t = D.require_cuda()
    if getattr(base, "kernel", "line") == "joseph":
        # Joseph weights exist in parity mode only: exact leaf factors + DGEMM
        # and the parity projector for the node systems
        gram, node_mode = "dense", "parity"
    depth = levels - 1
    p = (n >> depth) ** 2
    all_paths = _leaf_paths(levels)
    n_leaf = len(all_paths)
    names = ["/".join(q) or "root" for q in all_paths]
    # Leaves are assembled, inverted and (optionally) packed in chunks of at
    # most ~8 GB of Grams, so the full dense Grams never coexist (config 4 at
    # 6 levels: 1024 leaves of 4096^2 = 137 GB dense, 69 GB packed inverses).
    chunk = max(1, min(n_leaf, (8 << 30) // max(1, p * p * 8)))
    use_packed = packed and p % 128 == 0
    # keep a copy of the Grams (API: coarse_solve.lower, a Cholesky factor
    # computed on first access) only when they are small; the V-cycle itself
    # only needs the inverses
    keep_gram = n_leaf * p * p * 8 <= (8 << 30)
    gram_copy = None
    inverses = None
    from .sparse_kernels import PackedSymmetric
    for c0 in range(0, n_leaf, chunk):
        cpaths = all_paths[c0:c0 + chunk]
        if sharded:
            # angle-sharded W: every rank accumulates its angles' share of each
            # leaf Gram (the Gram is a sum over rays), one NCCL allreduce sums
            # them, and every rank inverts all leaves (coarse solves are local)
            _, grams = _assemble_leaf_grams(base, n, 0.0, levels, paths=cpaths, method=gram,
                                            full=False)
            w.dist.all_reduce(grams, group=w.group)
            if lam != 0:
                grams.diagonal(dim1=1, dim2=2).add_(lam)
        else:
            _, grams = _assemble_leaf_grams(w, n, lam, levels, paths=cpaths, method=gram,
                                            full=False)
        if keep_gram:
            if gram_copy is None:
                gram_copy = t.empty((n_leaf, p, p), dtype=t.float64, device=grams.device)
            gram_copy[c0:c0 + len(cpaths)].copy_(grams)
        sub = 4 << 30
        batch = max(1, min(len(cpaths), sub // max(1, p * p * 8)))
        for b0 in range(0, len(cpaths), batch):
            try:
                # hand-written batched SPD inverse on the fp64 tensor cores (in place)
                spd_inverse_(grams[b0:b0 + batch], names=names[c0 + b0:c0 + b0 + batch])
            except NotPositiveDefiniteError as exc:
                name, _, why = str(exc).partition(": ")
                raise NotPositiveDefiniteError(
                    f"coarsest subproblem '{name}' is singular (lambda={lam}): {why}") from None
        if use_packed:
            # packed symmetric storage: the V-cycle's coarse solves stream half the bytes
            pk = PackedSymmetric.pack(grams)
            if inverses is None:
                inverses = PackedSymmetric(
                    t.empty((n_leaf, pk.data.shape[1]), dtype=t.float64, device=grams.device), p)
            inverses.data[c0:c0 + len(cpaths)].copy_(pk.data)
            del pk
        else:
            if inverses is None:
                inverses = t.empty((n_leaf, p, p), dtype=t.float64, device=grams.device)
            inverses[c0:c0 + len(cpaths)].copy_(grams)
        del grams
    paths = all_paths
    leaf_index = {path: i for i, path in enumerate(paths)}
    if node_mode not in ("fast", "fast32", "parity"):
        raise ValueError(f"unknown node_mode '{node_mode}'")
    from .geometry import LineProjector
    if node_mode == "parity" or (node_mode == "fast" and getattr(base, "mode", None) == "fast"
                                 and getattr(base, "precision", None) == N.F64):
        node_w = w
    elif sharded:
        # node systems on the same angle shards: pair per rank + allreduce of W^T y
        from .sharding import AngleShardedProjector
        node_w = AngleShardedProjector(
            w.geometry, group=w.group, precision="float64" if node_mode == "fast" else "float32",
            mode="fast", scheme=w.scheme, device=w.device, always_reduce=w.collectives)
    elif node_mode == "fast":
        node_w = LineProjector(w.geometry, precision="float64", mode="fast", device=w.device)
    else:
        node_w = LineProjector(w.geometry, precision="float32", mode="fast", device=w.device)

    def make(bands, level):
        side = n >> (level - 1)
        path = "/".join(bands)
        if level == levels:
            li = leaf_index[bands]
            return WmgNode(side=side, level=level, path=path, factor=None, lam=lam,
                           coarse_solve=DenseFactorization(
                               dimension=p, inverse=inverses[li],
                               gram=None if gram_copy is None else gram_copy[li]),
                           bands=bands)
        node = WmgNode(side=side, level=level, path=path, factor=w, lam=lam,
                       intergrid=None, bands=bands)
        for b in BAND_IDS:
            node.children[b] = make(bands + (b,), level + 1)
        return node

    root = make((), 1)
    h = WmgHierarchy(levels=levels, lam=lam, root=root, projector=w, n=n, nu_pre=nu_pre,
                     nu_post=nu_post, leaf_factors=None, leaf_inverses=inverses,
                     node_projector=node_w)
    for nd in h.nodes():
        nd.hierarchy = h
        if not nd.is_coarsest:
            nd.intergrid = _LazyIntergrid(nd.side)
    if nu_pre or nu_post:
        _setup_smoothers(h)
    return h


class _LazyIntergrid:
    """Host CSR intergrid set built on first access (API compatibility only)."""

    def __init__(self, side):
        self.n = side
        self._set = None

    def __getitem__(self, band):
        if self._set is None:
            self._set = build_intergrid_set(self.n)
        return self._set[band]


def smoother_start_vector(dim: int) -> np.ndarray:
    """Fixed, positive start vector of the smoother's power iteration:
    v_i = 1 + ((7919 i) mod 1013) / 1013 (integer arithmetic and one IEEE
    division -- identical on every host)."""
    i = np.arange(dim, dtype=np.int64)
    return 1.0 + ((i * 7919) % 1013).astype(np.float64) / 1013.0


def smoother_scaling(colsum_host: np.ndarray, n: int, depth: int) -> np.ndarray:
    """C_p of a node at band-path depth k: 1 / (2^-k * the sum of W's column
    sums over each 2^k x 2^k block of fine pixels), zero sums -> 0 (the SIRT
    convention of solvers.py:84-85).  Host numpy, so the result is bitwise the
    same wherever it is evaluated."""
    B = 1 << depth
    blk = colsum_host.reshape(n // B, B, n // B, B).sum(axis=(1, 3)).reshape(-1)
    blk = blk * (0.5 ** depth)
    with np.errstate(divide="ignore"):
        return np.where(blk > 0, 1.0 / blk, 0.0)


def _setup_smoothers(h: WmgHierarchy, power_iterations: int = 10):
    """C_p and omega_p = 0.95 / lambda_max(C_p A_p) for the SIRT-type node
    smoother (module docstring).  Deterministic: C_p from the column sums (bit-
    identical to the reference's W^T 1) summed on the host, lambda_max from
    ``power_iterations`` steps from ``smoother_start_vector`` with DET_SUM norms
    and dots (oracle/multilevel.py restates the same procedure)."""
    t = D.torch()
    w = h.projector
    colsum = w.col_sums_dev().cpu().numpy()
    for nd in h.nodes():
        if nd.is_coarsest:
            continue
        k = len(nd.bands)
        c = t.from_numpy(smoother_scaling(colsum, h.n, k)).to(w.device)
        nd.smooth_c = c.contiguous()
        v = t.from_numpy(smoother_start_vector(nd.dim)).to(w.device)
        out = t.empty_like(v)
        lam = None
        for _ in range(power_iterations):
            nrm = D.det_norm_sq(v).sqrt_()
            v = v / nrm
            nd.apply_system_(v, out)
            out.mul_(c)
            lam = D.det_dot(v, out)            # stays on the device: one read at the end
            v = out.clone()
        lam_max = float(lam.item()) if lam is not None else 1.0
        nd.smooth_omega = 0.95 / lam_max if lam_max > 0 else 0.0


# ------------------------------------------------------------------ V-cycle
def _node_solve_(node: WmgNode, r, multiplicative: bool):
    """Approximate solve of the node system (device tensors)."""
    if node.is_coarsest:
        return node.coarse_solve.apply_inverse(r)
    h = node.hierarchy
    if h is None or (h.nu_pre == 0 and h.nu_post == 0):
        return _wtg_(node, r, multiplicative)
    t = D.torch()
    z = t.zeros_like(r)
    az = t.empty_like(r)
    res = t.empty_like(r)

    def sweep(z_is_zero):
        # z += omega C (r - A z), one fused kernel (same rounding as the unfused form)
        if z_is_zero:
            D.smooth_update(z, node.smooth_omega, node.smooth_c, r)
        else:
            node.apply_system_(z, az)
            D.smooth_update(z, node.smooth_omega, node.smooth_c, r, az)

    zero = True
    for _ in range(h.nu_pre):
        sweep(zero)
        zero = False
    if zero:
        e = _wtg_(node, r, multiplicative)
        z.copy_(e)
    else:
        node.apply_system_(z, az)
        D.axpy(res, r, 1.0, -1, az)
        e = _wtg_(node, res, multiplicative)
        D.axpy(z, z, 1.0, +1, e)
    for _ in range(h.nu_post):
        sweep(False)
    return z


# ------------------------------------------------ sibling batches (hybrid cycle)
# In the hybrid cycle the LH/HL/HH children of a node are solved independently,
# so nodes of one depth are processed in lockstep: one batched projector pair
# serves all their node-system applications (on small grids one launch of the
# batched fp64 kernels instead of one per node).  Every item is computed
# exactly as by the single-node path (same kernels, same arithmetic), so the
# batched cycle is bit-identical to the sequential one.
BATCH_SIBLINGS = True      # tests switch it off to compare with the sequential cycle


def _batchable(h) -> bool:
    w = h.node_projector
    return BATCH_SIBLINGS and hasattr(w, "forward_batch_") and not _is_sharded(w)


def _apply_system_batch_(nodes, V, OUT):
    """OUT[b] = (P_b^T P_b + lam) V[b] for nodes of one depth (batched pair)."""
    h = nodes[0].hierarchy
    w = h.node_projector
    B = len(nodes)
    k = len(nodes[0].bands)
    n2 = h.n * h.n
    M = w.shape[0]
    fused = FUSED_PATHS and k > 0 and V.is_contiguous() and OUT.is_contiguous()
    sino = h.buf(("bsino", B), B * M).view(B, M)
    if fused and getattr(w, "supports_forward_path", False):
        # prolongation evaluated inside the forward's padding pass
        w.forward_path_(V, [nd.bands for nd in nodes], sino)
    else:
        F = h.buf(("bpf", B), B * n2).view(B, n2)
        if fused:
            prolong_path(h.n, [nd.bands for nd in nodes], V, F)
        else:
            for b, nd in enumerate(nodes):
                cur = V[b]
                for lv in range(k - 1, -1, -1):
                    side_f = h.n >> lv
                    dst = F[b] if lv == 0 else h.buf(("bpfl", lv, b), side_f * side_f)
                    prolong(side_f, cur, nd.bands[lv], dst, accumulate=False)
                    cur = dst
        w.forward_batch_(F, sino)
    img = h.buf(("bimg", B), B * n2).view(B, n2)
    w.backward_batch_(sino, img)
    if fused:
        restrict_path(h.n, [nd.bands for nd in nodes], img, OUT)
    for b, nd in enumerate(nodes):
        cur = img[b]
        for lv in range(k if not fused else 0):
            side_f = h.n >> lv
            dst = OUT[b] if lv == k - 1 else h.buf(("brs", lv, b), (side_f // 2) ** 2)
            restrict(side_f, cur, (nd.bands[lv],), out=dst.view(1, -1))
            cur = dst
        if nd.lam != 0:
            D.add_scaled(OUT[b], OUT[b], nd.lam, +1, V[b])
    return OUT


def _leaf_solve_batch_(nodes, R, Z):
    """Z[b] = G_b^-1 R[b]: one batched GEMV per run of consecutive leaf slots."""
    h = nodes[0].hierarchy
    slots = [_leaf_slot(h, nd) for nd in nodes]
    from .sparse_kernels import batched_gemv
    i = 0
    while i < len(slots):
        j = i + 1
        while j < len(slots) and slots[j] == slots[j - 1] + 1:
            j += 1
        batched_gemv(h.leaf_inverses[slots[i]:slots[i] + (j - i)], R[i:j], out=Z[i:j])
        i = j
    return Z


def _node_solve_batch_(nodes, R):
    """Z[b] ~= A_b^-1 R[b] for hybrid-cycle nodes of one depth (R: (B, dim))."""
    t = D.torch()
    B = len(nodes)
    if B == 1:
        return _node_solve_(nodes[0], R[0].contiguous(), False).view(1, -1)
    h = nodes[0].hierarchy
    if nodes[0].is_coarsest:
        if h is not None and h.leaf_inverses is not None:
            return _leaf_solve_batch_(nodes, R, t.empty_like(R))
        return t.stack([_node_solve_(nd, R[b].contiguous(), False)
                        for b, nd in enumerate(nodes)])
    if h.nu_pre == 0 and h.nu_post == 0:
        return _wtg_batch_(nodes, R)
    R = R.contiguous()
    Z = t.zeros_like(R)
    AZ = t.empty_like(R)
    RES = t.empty_like(R)
    omegas = [nd.smooth_omega for nd in nodes]
    scalings = [nd.smooth_c for nd in nodes]

    def sweep(z_is_zero):
        if not z_is_zero:
            _apply_system_batch_(nodes, Z, AZ)
        D.smooth_update_batch(Z, omegas, scalings, R, None if z_is_zero else AZ)

    zero = True
    for _ in range(h.nu_pre):
        sweep(zero)
        zero = False
    if zero:
        Z.copy_(_wtg_batch_(nodes, R))
    else:
        _apply_system_batch_(nodes, Z, AZ)
        D.axpy(RES.view(-1), R.view(-1), 1.0, -1, AZ.view(-1))
        E = _wtg_batch_(nodes, RES)
        D.axpy(Z.view(-1), Z.view(-1), 1.0, +1, E.view(-1))
    for _ in range(h.nu_post):
        sweep(False)
    return Z


def _wtg_batch_(nodes, R):
    """Hybrid two-grid correction of several nodes of one depth in lockstep."""
    t = D.torch()
    B = len(nodes)
    side = nodes[0].side
    nc = (side // 2) ** 2
    R = R.contiguous()
    RLL = t.empty((B, nc), dtype=R.dtype, device=R.device)
    restrict_batch(side, R, ("LL",), RLL)
    ZLL = _node_solve_batch_([nd.children["LL"] for nd in nodes], RLL).contiguous()
    E = t.empty_like(R)
    prolong_batch(side, ZLL, ("LL",), E, accumulate=False)
    AE = t.empty_like(R)
    _apply_system_batch_(nodes, E, AE)
    RW = t.empty_like(R)
    D.axpy(RW.view(-1), R.view(-1), 1.0, -1, AE.view(-1))
    RB = t.empty((B, 3, nc), dtype=R.dtype, device=R.device)
    restrict_batch(side, RW, ("LH", "HL", "HH"), RB)
    kids = [nd.children[band] for nd in nodes for band in ("LH", "HL", "HH")]
    ZK = _node_solve_batch_(kids, RB.view(3 * B, nc)).contiguous()
    prolong_batch(side, ZK, ("LH", "HL", "HH"), E, accumulate=True)
    return E


def _wtg_(node: WmgNode, r, multiplicative: bool):
    """One wavelet two-grid correction, zero initial guess (multilevel.py:175-198)."""
    t = D.torch()
    side = node.side
    r_ll = restrict(side, r, ("LL",))[0]
    e = t.empty_like(r)
    prolong(side, _node_solve_(node.children["LL"], r_ll, multiplicative), "LL", e,
            accumulate=False)
    ae = t.empty_like(r)
    r_work = t.empty_like(r)
    node.apply_system_(e, ae)
    D.axpy(r_work, r, 1.0, -1, ae)
    if not multiplicative:
        rb = restrict(side, r_work, ("LH", "HL", "HH"))
        kids = [node.children[b] for b in ("LH", "HL", "HH")]
        h = node.hierarchy
        if all(k.is_coarsest for k in kids) and h is not None and h.leaf_inverses is not None:
            # the three sibling leaves are consecutive in the leaf tensor
            i0 = _leaf_slot(h, kids[0])
            from .sparse_kernels import batched_gemv
            zb3 = batched_gemv(h.leaf_inverses[i0:i0 + 3], rb)
            for i, band in enumerate(("LH", "HL", "HH")):
                prolong(side, zb3[i], band, e, accumulate=True)
            return e
        if h is not None and _batchable(h):
            zk = _node_solve_batch_(kids, rb)          # the three siblings in lockstep
            for i, band in enumerate(("LH", "HL", "HH")):
                prolong(side, zk[i], band, e, accumulate=True)
            return e
        for i, band in enumerate(("LH", "HL", "HH")):
            zb = _node_solve_(kids[i], rb[i].contiguous(), multiplicative)
            prolong(side, zb, band, e, accumulate=True)
        return e
    for band in ("LH", "HL", "HH"):
        r_band = restrict(side, r_work, (band,))[0]
        zb = _node_solve_(node.children[band], r_band, multiplicative)
        prolong(side, zb, band, e, accumulate=True)
        if band != "HH":
            node.apply_system_(e, ae)
            D.axpy(r_work, r, 1.0, -1, ae)
    return e


def _leaf_slot(h, leaf):
    """Index of a leaf in the hierarchy's leaf tensors (paths in band order)."""
    idx = 0
    for b in leaf.bands:
        idx = idx * 4 + BAND_CODE[b]
    return idx


def wtg_apply(node: WmgNode, r, multiplicative: bool = False):
    """One wavelet two-grid correction for the node's system, zero initial guess."""
    rd, was_np = D.to_device(r)
    if rd.numel() != node.dim:
        raise DimensionMismatchError(f"wtg_apply: residual length {rd.numel()} != {node.dim}")
    if node.is_coarsest:
        raise ValueError("wtg_apply needs an internal node")
    return D.to_caller(_wtg_(node, rd, multiplicative), was_np)


class _GraphedOperator:
    """Device operator whose eager body has no data-dependent control flow: after
    one eager warm-up it is captured once as a CUDA graph (static input/output
    buffers) and replayed, so its ~50-300 small launches cost one graph launch."""

    _wmg_device = True
    dim = 0

    def _init_graph(self, graph: bool):
        self.use_graph = graph
        self._graph = None
        self._gin = self._gout = None
        self._eager_calls = 0

    def _eager(self, v):  # pragma: no cover - abstract
        raise NotImplementedError

    def prepare(self):
        """Warm up and capture the graph now (part of the setup), so the first
        solve replays instead of capturing."""
        if self.use_graph and self._graph is None:
            t = D.torch()
            z = t.zeros(self.dim, dtype=t.float64, device=self._device())
            out = t.empty_like(z)
            while self._graph is None and self.use_graph:
                self.apply_(z, out)
        return self

    def _device(self):  # pragma: no cover - overridden
        raise NotImplementedError

    def apply_(self, v, out):
        t = D.torch()
        if not self.use_graph:
            out.copy_(self._eager(v))
            return out
        if self._graph is None:
            if self._eager_calls < 1:               # warm-up (allocator, buffers)
                self._eager_calls += 1
                out.copy_(self._eager(v))
                return out
            self._gin = t.empty_like(v)
            self._gin.copy_(v)
            try:
                g, self._gout = D.capture_graph(lambda: self._eager(self._gin), v.device)
            except RuntimeError as exc:
                if not getattr(self, "_sharded", False):
                    raise
                # a collective the communicator cannot capture: keep this rank's
                # cycle eager (the sequence of collectives is unchanged)
                import warnings
                warnings.warn(f"sharded V-cycle not captured, running eagerly: {exc}")
                self.use_graph = False
                out.copy_(self._eager(v))
                return out
            self._graph = g
        self._gin.copy_(v)
        self._graph.replay()
        out.copy_(self._gout)
        return out

    def __call__(self, v):
        t = D.torch()
        vd, was_np = D.to_device(v)
        if vd.numel() != self.dim:
            raise DimensionMismatchError(
                f"{type(self).__name__}: length {vd.numel()} != {self.dim}")
        out = t.empty_like(vd)
        self.apply_(vd, out)
        return D.to_caller(out, was_np)


class WmgPreconditioner(_GraphedOperator):
    """One V-cycle as an approximate solve of (W^T W + lam I) z = v."""

    def __init__(self, h: WmgHierarchy, multiplicative: bool = False, graph: bool = True):
        self.h = h
        self.multiplicative = multiplicative
        self.dim = h.root.dim
        # an angle-sharded cycle runs collectives between its kernels: captured
        # with them when they are NCCL's (stream-ordered), eager over gloo
        self._sharded = _is_sharded(h.node_projector)
        self._init_graph(graph and (not self._sharded or
                                    getattr(h.node_projector, "graph_capturable", False)))

    def _eager(self, v):
        return _node_solve_(self.h.root, v, self.multiplicative)

    def _device(self):
        return self.h.projector.device


def wmg_preconditioner(h: WmgHierarchy, multiplicative: bool = False,
                       graph: bool = True) -> Callable:
    """One V-cycle as the preconditioner (multilevel.py:201-208); with
    ``graph`` the cycle is captured as a CUDA graph here, in the setup."""
    return WmgPreconditioner(h, multiplicative, graph=graph).prepare()


# --------------------------------------------- classical two-grid
class ClassicalTGPreconditioner(_GraphedOperator):
    """One classical two-grid cycle on the normal equations, LL coarsening only
    (multilevel.py:211-258).  Smoother (the reference's, applied verbatim):
    z <- z + C (v - (W^T R W + lam) z); coarse correction with the dense
    Galerkin operator of W^T W + lam I under the LL restriction (exact weights,
    stored inverse, our batched GEMV)."""

    _wmg_device = True

    def __init__(self, w, n: int, lam: float, smoother_steps=(1, 1), graph: bool = True):
        _check_even(n)
        nu1, nu2 = smoother_steps
        if nu1 < 0 or nu2 < 0:
            raise ValueError("smoothing counts must be nonnegative")
        if w.shape[1] != n * n:
            raise DimensionMismatchError(
                f"projector has {w.shape[1]} columns, expected {n * n}")
        if not hasattr(w, "handle"):
            raise TypeError("classical_tg_preconditioner needs a LineProjector")
        t = D.require_cuda()
        from .solvers import sirt_scaling
        self.w, self.n, self.lam = w, n, float(lam)
        self.nu1, self.nu2 = int(nu1), int(nu2)
        sc = sirt_scaling(w)
        self.c, self.r = sc.c_dev, sc.r_dev
        _, grams = _assemble_leaf_grams(
            w, n, lam, 2, paths=[("LL",)], full=False,
            method="dense" if getattr(w, "kernel", "line") == "joseph" else "sparse")
        gram = grams[0].clone() if grams[0].numel() * 8 <= (2 << 30) else None
        try:
            spd_inverse_(grams)
        except NotPositiveDefiniteError:
            raise NotPositiveDefiniteError(
                f"coarse LL Galerkin operator is singular (lambda={lam})") from None
        inv = grams[0]
        if inv.shape[-1] % 128 == 0:
            from .sparse_kernels import PackedSymmetric
            inv = PackedSymmetric.pack(grams)
            del grams
        self.coarse = DenseFactorization(dimension=inv.shape[-1], inverse=inv, gram=gram)
        M, N_ = w.shape
        dev = w.device
        self._sino = t.empty(M, dtype=t.float64, device=dev)
        self._img = t.empty(N_, dtype=t.float64, device=dev)
        self.dim = n * n
        self._init_graph(graph)

    def _apply_a(self, v, out):
        self.w.forward_(v, self._sino)
        self.w.backward_(self._sino, out)
        if self.lam != 0:
            D.add_scaled(out, out, self.lam, +1, v)
        return out

    def _smooth(self, z, v):
        t = D.torch()
        self.w.forward_(z, self._sino)
        D.hadamard(self._sino, self.r, self._sino)          # r * (W z)
        self.w.backward_(self._sino, self._img)             # W^T (r * W z)
        D.add_scaled(self._img, self._img, self.lam, +1, z)  # + lam z
        u = t.empty_like(v)
        D.axpy(u, v, 1.0, -1, self._img)                    # v - (...)
        D.hadamard(u, self.c, u)                            # C (...)
        D.axpy(z, z, 1.0, +1, u)                            # z + C(...)
        return z

    def _device(self):
        return self.w.device

    def _eager(self, v):
        t = D.torch()
        z = t.zeros_like(v)
        for _ in range(self.nu1):
            self._smooth(z, v)
        if self.nu1 > 0:
            az = t.empty_like(v)
            self._apply_a(z, az)
            res = t.empty_like(v)
            D.axpy(res, v, 1.0, -1, az)
        else:
            res = v
        rc = restrict(self.n, res, ("LL",))[0]
        zc = self.coarse.apply_inverse(rc)
        prolong(self.n, zc, "LL", z, accumulate=True)
        for _ in range(self.nu2):
            self._smooth(z, v)
        return z



def classical_tg_preconditioner(w, n: int, lam: float, smoother_steps=(1, 1),
                                graph: bool = True) -> Callable:
    return ClassicalTGPreconditioner(w, n, lam, smoother_steps, graph=graph).prepare()
