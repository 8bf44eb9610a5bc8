"""Angle-sharded WMG-CGLS (SURVEY.md s8 row e): two ranks (gloo, both on the
one GPU of the test box -- no kernel waits on another rank's kernel; the
collectives are host-side) each own the mirror shard of the angles.  Leaf
Grams are per-rank partial sums + allreduce, node systems are sharded pairs +
allreduce of W^T y, the Krylov vectors are replicated.  The result must match
the single-rank solve (same algorithm, reordered sums) to 1e-8 with the same
iteration count."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N_, D_, M_ = 64, 91, 90


def _problem():
    from paper_1310_0956_b200 import build_geometry, build_projector, random_ellipses
    g = build_geometry(N_, D_, M_)
    x_ex = random_ellipses(N_, 10, seed=0)
    b = build_projector(g) @ x_ex
    return g, b


def _solve(w, g, b, lam, levels, nu):
    from paper_1310_0956_b200 import (SolverConfig, build_wmg_hierarchy, cgls_solve,
                                      wmg_preconditioner)
    h = build_wmg_hierarchy(w, N_, lam, levels, nu_pre=nu, nu_post=nu)
    cfg = SolverConfig(max_iterations=40, residual_tolerance=1e-5, regularization_lambda=lam)
    return cgls_solve(w, b, precond=wmg_preconditioner(h), cfg=cfg)


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1310_0956_b200.sharding import AngleShardedProjector
        g, b = _problem()
        out = []
        for lam, levels, nu in ((1e-3, 3, 0), (0.0, 2, 2)):
            w = AngleShardedProjector(g, precision="float64", mode="fast", device="cuda:0")
            bl = w.scatter_sinogram(torch.from_numpy(b).cuda())
            x, rec = _solve(w, g, bl, lam, levels, nu)
            out.append((x.cpu().numpy(), rec.iterations[-1], rec.status))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_sharded_wmg_cgls_matches_single_rank(gpu):
    import torch.multiprocessing as mp
    from paper_1310_0956_b200 import build_projector
    g, b = _problem()
    ref = []
    for lam, levels, nu in ((1e-3, 3, 0), (0.0, 2, 2)):
        w = build_projector(g, precision="float64", mode="fast")
        x, rec = _solve(w, g, b, lam, levels, nu)
        ref.append((x, rec.iterations[-1], rec.status))
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = 2
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, out in res:
        for (x, it, st), (xr, itr, str_) in zip(out, ref):
            assert st == str_
            assert abs(it - itr) <= 1
            assert np.linalg.norm(x - xr) <= 1e-8 * np.linalg.norm(xr), rank
    np.testing.assert_array_equal(res[0][1][0][0], res[1][1][0][0])   # replicas agree
