"""Multi-rank host logic on CPU: world size 2, gloo backend, 127.0.0.1.

The rank-local projector is a CPU stand-in built from the pinned oracle CSR of
the rank's angles (test-only); the sharding layer (angle partition, summed
backprojection, sinogram scatter/gather, scalar reductions) is the product
code in paper_1310_0956_b200/sharding.py.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1310_0956_b200.sharding import (angle_weights, shard_angles, shard_slices)


def test_partitions_cover_and_balance():
    m = 720
    for world in (1, 2, 4, 8):
        rr = [shard_angles(m, world, r) for r in range(world)]
        assert np.array_equal(np.sort(np.concatenate(rr)), np.arange(m))
        a = np.arange(m) * (np.pi / m)
        w = angle_weights(a)
        loads = np.array([w[ix].sum() for ix in rr])
        assert loads.max() / loads.mean() < 1.01           # round robin is balanced
        cont = [shard_angles(m, world, r, "contiguous") for r in range(world)]
        assert np.array_equal(np.concatenate(cont), np.arange(m))
        sl = [shard_slices(256, world, r) for r in range(world)]
        assert np.array_equal(np.concatenate(sl), np.arange(256))
    with pytest.raises(ValueError):
        shard_angles(10, 2, 2)


@pytest.mark.parametrize("m", [90, 180, 720, 4096, 7, 1, 2])
def test_mirror_shards_closed_and_balanced(m):
    """The "mirror" scheme partitions the angles, every shard is closed under
    k -> m - k (so it keeps the symmetric kernels) and work is balanced."""
    a = np.arange(m) * (np.pi / m)
    w = angle_weights(a)
    for world in (1, 2, 3, 4, 8):
        sh = [shard_angles(m, world, r, "mirror") for r in range(world)]
        assert np.array_equal(np.sort(np.concatenate(sh)), np.arange(m))
        for ix in sh:
            assert np.all(np.diff(ix) > 0)
            s = set(ix.tolist())
            assert all((m - k) in s for k in s if k != 0 and 2 * k != m)
        if m >= 90 * world:
            loads = np.array([w[ix].sum() for ix in sh])
            assert loads.max() / loads.mean() < 1.02


@pytest.mark.parametrize("m", [180, 720, 4096, 8, 4, 90, 7])
def test_quad_shards_closed_and_balanced(m):
    """The "quad" scheme (AngleShardedProjector's default) partitions the
    angles into shards closed under the mirror k -> m - k AND the transposition
    theta -> pi/2 -+ theta (k -> m/2 - k, or 3m/2 - k past pi/2), so ranks keep
    the eight-image backprojector; m % 4 != 0 falls back to the mirror scheme."""
    a = np.arange(m) * (np.pi / m)
    w = angle_weights(a)
    for world in (1, 2, 3, 4, 8):
        sh = [shard_angles(m, world, r, "quad") for r in range(world)]
        assert np.array_equal(np.sort(np.concatenate(sh)), np.arange(m))
        if m % 4:
            assert all(np.array_equal(x, shard_angles(m, world, r, "mirror"))
                       for r, x in enumerate(sh))
            continue
        for ix in sh:
            s = set(ix.tolist())
            assert all((m - k) in s for k in s if k != 0 and 2 * k != m)
            for k in s:
                if k in (0, m // 2):
                    continue
                t = m // 2 - k if k < m // 2 else 3 * m // 2 - k
                assert t in s, (m, world, k)
        if m >= 180 * world:
            loads = np.array([w[ix].sum() for ix in sh])
            assert loads.max() / loads.mean() < 1.03


class _CpuLocal:
    """CPU stand-in for a rank-local LineProjector (oracle CSR of its angles)."""

    def __init__(self, n, d, angles):
        from oracle import cproj
        self.w = cproj.build_csr(n, d, angles)
        self.shape = self.w.shape

    def forward_(self, x, out):
        out.copy_(torch.from_numpy(self.w @ x.numpy()))
        return out

    def backward_(self, y, out):
        out.copy_(torch.from_numpy(self.w.T @ y.numpy()))
        return out


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1310_0956_b200.geometry import Geometry
        from paper_1310_0956_b200.sharding import AngleShardedProjector
        n, d, m = 32, 47, 30
        angles = np.arange(m) * (np.pi / m)
        g = Geometry(n, d, m, angles=angles)
        idx = shard_angles(m, world, rank, "mirror")
        sp = AngleShardedProjector(g, local=_CpuLocal(n, d, angles[idx]))
        rs = np.random.default_rng(0)
        x = torch.from_numpy(rs.standard_normal(n * n))
        y_full = torch.from_numpy(rs.standard_normal(m * d))
        y_loc = sp.scatter_sinogram(y_full)
        out = torch.empty(n * n, dtype=torch.float64)
        sp.backward_(y_loc, out)
        fx = torch.empty(sp.shape[0], dtype=torch.float64)
        sp.forward_(x, fx)
        full_fx = sp.gather_sinogram(fx)
        part = torch.tensor([float((fx * fx).sum())], dtype=torch.float64)
        sp.reduce_sino_(part)
        q.put((rank, out.numpy(), full_fx.numpy(), float(part[0])))
    finally:
        dist.destroy_process_group()


def test_angle_sharded_pair_world2():
    from oracle import cproj
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = 2
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n, d, m = 32, 47, 30
    angles = np.arange(m) * (np.pi / m)
    w = cproj.build_csr(n, d, angles)
    rs = np.random.default_rng(0)
    x = rs.standard_normal(n * n)
    y = rs.standard_normal(m * d)
    ref_b = w.T @ y
    ref_f = w @ x
    for rank, out, full_fx, nsq in res:
        # partition of the angle sum changes the order: 1e-15-level differences
        assert np.linalg.norm(out - ref_b) <= 1e-14 * np.linalg.norm(ref_b)
        assert np.array_equal(full_fx, ref_f)                  # rows are exact
        assert abs(nsq - float(ref_f @ ref_f)) <= 1e-12 * float(ref_f @ ref_f)
    np.testing.assert_array_equal(res[0][1], res[1][1])        # replicas agree
