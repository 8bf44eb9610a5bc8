"""Banded backprojection (wmg_backward_band) and the sharded W^T y whose
allreduce overlaps the remaining bands (sharding.AngleShardedProjector).

* one rank: the bands issued in order reproduce wmg_backward bit for bit
  (full config-3 geometry at n = 2048 and a quad shard of it);
* two ranks (gloo, both on cuda:0 -- host-side collectives, no kernel waits on
  another rank): the overlapped sharded W^T y equals the non-overlapped one bit
  for bit and the single-rank W^T y within fp32 summation-order rounding.
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world,rank", [(1, 0), (4, 1)])
def test_bands_bitwise(gpu, world, rank):
    torch = gpu
    from paper_1310_0956_b200.geometry import build_geometry, build_projector
    from paper_1310_0956_b200.sharding import shard_angles
    n, d, m = 2048, 2897, 2048
    g = build_geometry(n, d, m)
    if world > 1:
        g = g.subset(shard_angles(m, world, rank, "quad"))
    w = build_projector(g, precision="float32")
    qt = w.backward_bands()
    assert qt == n // 64
    y = torch.rand(w.shape[0], device="cuda")
    ref = torch.empty(n * n, device="cuda")
    w.backward_(y, ref)
    out = torch.full((n * n,), float("nan"), device="cuda")
    bounds = [0, 3, 10, 11, qt]
    for s0, s1 in zip(bounds[:-1], bounds[1:]):
        w.backward_band_(y, out, s0, s1)
        torch.cuda.synchronize()
        # rows of finished bands (top and mirrored bottom) are final; later
        # row-blocks hold only some of their tiles so far
        o, r = out.view(n, n), ref.view(n, n)
        assert torch.equal(o[: 32 * s1], r[: 32 * s1])
        assert torch.equal(o[n - 32 * s1:], r[n - 32 * s1:])
        if s1 < qt:
            assert torch.isnan(o[32 * s1: n - 32 * s1]).any()
    assert torch.equal(out, ref)


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_1310_0956_b200.geometry import build_geometry
    from paper_1310_0956_b200.sharding import AngleShardedProjector
    n, d, m = 2048, 2897, 2048
    g = build_geometry(n, d, m)
    w = AngleShardedProjector(g, precision="float32", device=torch.device("cuda", 0))
    yf = torch.from_numpy(np.random.default_rng(5).uniform(0, 1, m * d).astype(np.float32))
    y = w.scatter_sinogram(yf.cuda())
    a = torch.empty(n * n, device="cuda")
    w.overlap_groups = 4
    w.backward_(y, a)                       # overlapped (banded) path
    w.overlap_groups = 1
    b = torch.empty(n * n, device="cuda")
    w.backward_(y, b)                       # one allreduce after the whole backprojection
    torch.cuda.synchronize()
    if rank == 0:
        q.put((bool(torch.equal(a, b)), a.cpu().numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_overlap_two_ranks(gpu):
    torch = gpu
    import torch.multiprocessing as mp
    from paper_1310_0956_b200.geometry import build_geometry, build_projector
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    same, got = q.get(timeout=600)
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    assert same
    n, d, m = 2048, 2897, 2048
    w = build_projector(build_geometry(n, d, m), precision="float32")
    yf = torch.from_numpy(np.random.default_rng(5).uniform(0, 1, m * d).astype(np.float32))
    ref = w.backward(yf.cuda()).cpu().numpy()
    assert np.linalg.norm(got - ref) <= 1e-6 * np.linalg.norm(ref)
