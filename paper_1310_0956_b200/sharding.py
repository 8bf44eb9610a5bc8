"""Multi-GPU decomposition of the hot path (one process per GPU).

SURVEY.md s8(e):
  * projector pair (configs 2/3): angles (sinogram rows) are partitioned across
    ranks, the image is replicated.  A x is rank-local; A^T y is a sum over
    angles, so each rank backprojects its own rows and the partial images are
    summed with ONE allreduce (NCCL over NVLink on the GPU box) -- the path's
    only exchange.  Sinogram-space inner products need a scalar allreduce.
  * slice stacks (config 4): independent slices are dealt to ranks; no
    collective on the data path.

Round-robin assignment (angle k -> rank k mod world) balances the per-angle
work (nnz per angle ~ |cos| + |sin|; contiguous blocks differ by up to 8 %).

``AngleShardedProjector`` wraps a rank-local projector (a ``LineProjector`` of
the rank's angles on the GPU; tests inject a CPU stand-in) and implements the
same operator protocol plus ``reduce_sino_`` for the solvers' sinogram dots.
"""
from __future__ import annotations

import numpy as np


def shard_angles(n_angles: int, world: int, rank: int, scheme: str = "round_robin"):
    """Indices of the angles owned by ``rank`` (ascending).

    "round_robin": angle k -> rank k mod world.  "contiguous": equal blocks.
    "mirror": the units {k, m - k} (mirror pairs theta, pi - theta of an
    equiangular set) and {0, m/2} (the axis angles) are dealt round-robin, so
    every shard is closed under the mirror and keeps the symmetric kernels
    (4 pixel/ray images per weight evaluation); units have equal work.
    "quad" (default of AngleShardedProjector): mirror-and-transposition
    closed units of four angles, see below."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    if scheme == "round_robin":
        return np.arange(rank, n_angles, world)
    if scheme == "quad":
        # units {k, m-k, m/2-k, m/2+k} (theta, pi - theta, pi/2 -+ theta), the
        # diagonal pair {m/4, 3m/4} and the axis pair {0, m/2}, dealt
        # round-robin: every shard is closed under the mirror AND the
        # transposition, so ranks keep the eight-image backprojector; equal work
        # per quad.  Needs m % 4 == 0 (else the mirror scheme).
        m = n_angles
        if m % 4 or m < 4:
            return shard_angles(n_angles, world, rank, "mirror")
        # Quads of 4 adjacent angles stay on one rank: the symmetric forward packs 4
        # adjacent angles into a warp, whose rays then read the same words -- with
        # single quads dealt round-robin a rank's angles are `world` steps apart
        # and its forward ran at 0.56 of the unsharded efficiency at world = 8,
        # n = 4096 (tools/probe_shard_eff.py).  Whole rounds of such chunks are
        # dealt round-robin; what is left (fewer than 4 world + 3 quads, the
        # diagonal pair and the axis pair) goes, heaviest first, to the lightest rank.
        def quad(k):
            return [k, m - k, m // 2 - k, m // 2 + k]

        ks = list(range(1, m // 4))
        nround = (len(ks) // 4 // world) * world          # chunks dealt in whole rounds
        shards = [[] for _ in range(world)]
        for c in range(nround):
            shards[c % world] += [a for k in ks[4 * c:4 * c + 4] for a in quad(k)]
        left = [quad(k) for k in ks[4 * nround:]] + [[m // 4, 3 * m // 4], [0, m // 2]]
        wt = lambda u: float(np.sum(angle_weights(np.asarray(u) * (np.pi / m))))  # noqa: E731
        load = [wt(sh) if sh else 0.0 for sh in shards]
        for u in sorted(left, key=lambda u: (-wt(u), u[0])):
            r = min(range(world), key=lambda i: (load[i], i))
            shards[r] += u
            load[r] += wt(u)
        return np.array(sorted(shards[rank]), dtype=np.int64)
    if scheme == "mirror":
        m = n_angles
        units = [[0] + ([m // 2] if m % 2 == 0 and m > 1 else [])]
        units += [[k, m - k] for k in range(1, (m + 1) // 2)]
        mine = [a for u in units[rank::world] for a in u]
        return np.array(sorted(mine), dtype=np.int64)
    if scheme == "contiguous":
        bounds = np.linspace(0, n_angles, world + 1).round().astype(int)
        return np.arange(bounds[rank], bounds[rank + 1])
    raise ValueError(f"unknown scheme '{scheme}'")


def shard_slices(n_slices: int, world: int, rank: int):
    """Contiguous block of slice indices for ``rank`` (config 4)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    bounds = np.linspace(0, n_slices, world + 1).round().astype(int)
    return np.arange(bounds[rank], bounds[rank + 1])


def angle_weights(angles) -> np.ndarray:
    """Relative work per angle (|cos| + |sin|, proportional to nnz per angle)."""
    a = np.asarray(angles, dtype=np.float64)
    return np.abs(np.cos(a)) + np.abs(np.sin(a))


class AngleShardedProjector:
    """W restricted to this rank's angles, with a summed backprojection."""

    def __init__(self, g, group=None, precision: str = "float32", mode=None,
                 scheme: str = "quad", local=None, device=None, always_reduce=None):
        import os
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        backend = dist.get_backend(group) if dist.is_initialized() else None
        # ``always_reduce`` issues the collectives at world size 1 too (they are
        # in-place no-ops there): the one-GPU test boxes exercise the NCCL calls,
        # their stream ordering and their CUDA-graph capture this way
        if always_reduce is None:
            always_reduce = os.environ.get("WMG_ALWAYS_REDUCE", "0") == "1"
        self.collectives = dist.is_initialized() and (self.world > 1 or bool(always_reduce))
        # NCCL collectives are stream-ordered device work and can be captured in
        # a CUDA graph; gloo's are host-side, so loops over gloo stay eager
        self.graph_capturable = (not self.collectives) or (
            backend == "nccl" and os.environ.get("WMG_SHARDED_GRAPHS", "1") == "1")
        self.geometry = g
        self.scheme = scheme
        self.index = shard_angles(g.n_angles, self.world, self.rank, scheme)
        if local is None:
            from .geometry import build_projector
            local = build_projector(g.subset(self.index), precision=precision, mode=mode,
                                    device=device)
        self.local = local
        self.shape = (local.shape[0], g.n_image)       # rank-local rows x full image
        self.global_shape = (g.n_data, g.n_image)
        self.n_detectors = g.n_detectors

    # rank-local sinogram rows <-> full sinogram
    def scatter_sinogram(self, full):
        """This rank's rows of a full (m*d) sinogram (host or device array)."""
        d = self.n_detectors
        if hasattr(full, "reshape") and not isinstance(full, np.ndarray):
            import torch
            idx = torch.as_tensor(self.index, device=full.device)
            return full.reshape(-1, d).index_select(0, idx).reshape(-1).contiguous()
        return np.ascontiguousarray(np.asarray(full).reshape(-1, d)[self.index].reshape(-1))

    def gather_sinogram(self, local):
        """Full sinogram from every rank's rows (allgather; rank order restored)."""
        import torch
        d = self.n_detectors
        m = self.geometry.n_angles
        if self.world == 1:
            return local
        counts = [len(shard_angles(m, self.world, r, self.scheme)) for r in range(self.world)]
        width = max(counts) * d
        buf = torch.zeros(width, dtype=local.dtype, device=local.device)
        buf[: local.numel()] = local
        parts = [torch.empty_like(buf) for _ in range(self.world)]
        self.dist.all_gather(parts, buf, group=self.group)
        out = torch.empty(m * d, dtype=local.dtype, device=local.device).view(m, d)
        for r in range(self.world):
            idx = torch.as_tensor(shard_angles(m, self.world, r, self.scheme),
                                  device=local.device)
            out.index_copy_(0, idx, parts[r][: counts[r] * d].view(-1, d))
        return out.reshape(-1)

    # operator protocol (device tensors)
    def forward_(self, x, out):
        return self.local.forward_(x, out)

    # W^T y can be summed over the ranks band by band while the backprojection of
    # the later bands still runs (``overlap_groups`` groups of quadrant row-
    # blocks of equal work; the eight-image fp32 path only).  Default 1: one
    # allreduce after the whole backprojection.  Running a rank's backprojection
    # in band groups has a price -- at n = 4096 a rank's 1.82 ms (world = 8)
    # becomes 1.98 ms in 2 groups and 2.12 ms in 4 (world = 2: 7.2 -> 7.9 -> 8.4 ms;
    # tools/probe_shard_bands.py) -- which is as much as the 64 MB NVLink
    # allreduce it would hide (~0.2-0.3 ms over NVSwitch at world = 8), and the
    # last group's allreduce stays exposed.  Set > 1 where the exchange is slower.
    overlap_groups = int(__import__("os").environ.get("WMG_OVERLAP_GROUPS", "1"))

    def _band_groups(self, qt):
        total = qt * (qt + 1) // 2
        bounds, s, done = [0], 0, 0
        for k in range(1, self.overlap_groups + 1):
            target = total * k // self.overlap_groups
            while s < qt and done < target:
                done += qt - s
                s += 1
            if s > bounds[-1]:
                bounds.append(s)
        return list(zip(bounds[:-1], bounds[1:]))

    def backward_(self, y, out, accumulate=False):
        if accumulate:
            raise ValueError("accumulate is not supported on a sharded backprojection")
        qt = self.local.backward_bands() if (self.collectives and self.overlap_groups > 1 and
                                             hasattr(self.local, "backward_bands")) else 0
        if qt == 0:
            self.local.backward_(y, out)
            if self.collectives:
                self.dist.all_reduce(out, group=self.group)
            return out
        import torch
        n = self.geometry.n_pixels_per_side
        cur = torch.cuda.current_stream(out.device)
        comm = getattr(self, "_comm", None)
        if comm is None:
            comm = self._comm = torch.cuda.Stream(device=out.device)
        for s0, s1 in self._band_groups(qt):
            self.local.backward_band_(y, out, s0, s1)
            comm.wait_stream(cur)
            with torch.cuda.stream(comm):
                top = out[32 * s0 * n:32 * s1 * n]
                bot = out[(n - 32 * s1) * n:(n - 32 * s0) * n]
                if (n - 32 * s1) == 32 * s1:            # the two bands meet at the centre
                    self.dist.all_reduce(out[32 * s0 * n:(n - 32 * s0) * n], group=self.group)
                else:
                    self.dist.all_reduce(top, group=self.group)
                    self.dist.all_reduce(bot, group=self.group)
        cur.wait_stream(comm)
        return out

    def row_sums_dev(self):
        return self.local.row_sums_dev()            # rows are rank-local

    def col_sums_dev(self):
        c = self.local.col_sums_dev().clone()       # column sums = sum over angles
        if self.collectives:
            self.dist.all_reduce(c, group=self.group)
        return c

    @property
    def device(self):
        return self.local.device

    # matrix protocol the reference solvers use (w @ x, w.T @ y), on this
    # rank's rows: x is replicated, y holds this rank's sinogram rows
    def __matmul__(self, x):
        from . import _device as D
        t = D.torch()
        xd, was_np = D.to_device(x, device=self.device)
        out = t.empty(self.shape[0], dtype=xd.dtype, device=self.device)
        self.forward_(xd.reshape(-1), out)
        return D.to_caller(out, was_np)

    @property
    def T(self):
        return _ShardedTranspose(self)

    def reduce_sino_(self, t):
        """Sum rank-local sinogram-space partial reductions (in place)."""
        if self.collectives:
            self.dist.all_reduce(t, group=self.group)
        return t


class _ShardedTranspose:
    """W^T of an AngleShardedProjector: local backprojection + allreduce."""

    def __init__(self, w):
        self._w = w
        self.shape = (w.shape[1], w.shape[0])

    def __matmul__(self, y):
        from . import _device as D
        t = D.torch()
        yd, was_np = D.to_device(y, device=self._w.device)
        out = t.empty(self.shape[0], dtype=yd.dtype, device=self._w.device)
        self._w.backward_(yd.reshape(-1), out)
        return D.to_caller(out, was_np)
