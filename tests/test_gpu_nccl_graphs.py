"""Angle-sharded solver loops captured in CUDA graphs together with their NCCL
collectives (SURVEY.md s8 row e).

The test boxes have one GPU, and NCCL cannot put two ranks on one device, so
this runs a ONE-rank NCCL process group with ``always_reduce=True``: every
collective of the sharded path (the banded allreduces of W^T y on their comm
stream, the scalar allreduce of the sinogram dot, the leaf-Gram allreduce) is
issued -- in-place no-ops at world size 1 -- and captured.  That pins the part
that can break: stream ordering of the comm stream inside the capture, NCCL
calls under ``capture_begin``, replays.  Because the collectives do not change
the data at world size 1, every result must equal the unsharded solve bit for
bit, and the captured loop must equal the eager one."""
import os
import socket
import subprocess
import sys
import textwrap

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = textwrap.dedent(r"""
    import os, sys
    import numpy as np
    import torch
    import torch.distributed as dist
    sys.path.insert(0, os.environ["WMG_ROOT"])
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1,
                            device_id=torch.device("cuda:0"))
    from paper_1310_0956_b200 import (SolverConfig, build_geometry, build_projector,
                                      build_wmg_hierarchy, cgls_solve, random_ellipses,
                                      wmg_preconditioner)
    from paper_1310_0956_b200 import _device as D
    from paper_1310_0956_b200.sharding import AngleShardedProjector

    n, d, m = 64, 91, 90
    g = build_geometry(n, d, m)
    x_ex = random_ellipses(n, 10, seed=0)
    w0 = build_projector(g, precision="float64", mode="fast")
    b = torch.from_numpy(w0 @ x_ex).cuda()

    ws = AngleShardedProjector(g, precision="float64", mode="fast", device="cuda:0",
                               always_reduce=True)
    assert ws.collectives and ws.graph_capturable and ws.world == 1

    # 1. plain CGLS (lam != 0: both scalar reductions), graphed sharded loop
    cfg = SolverConfig(max_iterations=25, residual_tolerance=0.0, regularization_lambda=1e-3)
    xr, rr = cgls_solve(w0, b, cfg=cfg)
    xs, rs = cgls_solve(ws, b, cfg=cfg)
    loop = next(iter(ws.__dict__["_cgls_graph_cache"].values()))["loop"]
    assert loop.graph is not None, "sharded CGLS iteration was not captured"
    assert torch.equal(xr, xs), "graphed sharded CGLS != unsharded"
    assert rr.rel_residual == rs.rel_residual
    xe, re_ = cgls_solve(ws, b, cfg=cfg, graph=False)
    assert torch.equal(xe, xs), "graphed sharded CGLS != eager sharded"
    xs2, _ = cgls_solve(ws, b, cfg=cfg)             # replay of the cached graph
    assert torch.equal(xs2, xs)

    # 2. WMG-CGLS, nu = 2 + 2, 3 levels: the V-cycle graph holds the allreduces
    for lam, levels, nu in ((1e-3, 3, 0), (0.0, 3, 2)):
        cfg = SolverConfig(max_iterations=12, residual_tolerance=1e-9,
                           regularization_lambda=lam)
        hr = build_wmg_hierarchy(w0, n, lam, levels, nu_pre=nu, nu_post=nu)
        xr, rr = cgls_solve(w0, b, precond=wmg_preconditioner(hr), cfg=cfg)
        hs = build_wmg_hierarchy(ws, n, lam, levels, nu_pre=nu, nu_post=nu)
        ps = wmg_preconditioner(hs)
        xs, rs = cgls_solve(ws, b, precond=ps, cfg=cfg)
        assert ps._graph is not None, "sharded V-cycle was not captured"
        assert rr.iterations[-1] == rs.iterations[-1]
        err = float((xr - xs).norm() / xr.norm())
        assert err <= 1e-12, ("sharded graphed WMG-CGLS vs unsharded", lam, nu, err)
        pe = wmg_preconditioner(hs, graph=False)
        xe, re_ = cgls_solve(ws, b, precond=pe, cfg=cfg, graph=False)
        assert torch.equal(xe, xs), "graphed sharded WMG-CGLS != eager sharded"

    # 3. fp32 eight-image backprojection in bands with the allreduces on the comm
    #    stream (the overlap path), captured and replayed
    n, d, m = 2048, 2897, 64          # banded (eight-image) path: n >= 1728
    g = build_geometry(n, d, m)
    wf = AngleShardedProjector(g, precision="float32", device="cuda:0", always_reduce=True)
    wf.overlap_groups = 4                             # the banded overlap path
    assert wf.local.backward_bands() > 0, "expected the banded eight-image path"
    y = torch.rand(m * d, device="cuda", dtype=torch.float32,
                   generator=torch.Generator("cuda").manual_seed(5))
    ref = torch.empty(n * n, device="cuda", dtype=torch.float32)
    wf.local.backward_(y, ref)
    out = torch.zeros_like(ref)
    wf.backward_(y, out)                              # eager (creates the comm stream)
    assert torch.equal(out, ref)
    out.zero_()
    graph, _ = D.capture_graph(lambda: wf.backward_(y, out), torch.device("cuda:0"))
    for _ in range(3):
        out.zero_()
        graph.replay()
        torch.cuda.synchronize()
        assert torch.equal(out, ref), "captured banded backprojection + allreduce"
    torch.cuda.synchronize()
    dist.destroy_process_group()
    print("NCCL-GRAPHS-OK")
""")


def test_sharded_loops_capture_nccl_collectives(gpu, tmp_path):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    script = tmp_path / "nccl_graph_worker.py"
    script.write_text(WORKER)
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WMG_ROOT=ROOT,
               NCCL_DEBUG="WARN")
    r = subprocess.run([sys.executable, str(script)], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "NCCL-GRAPHS-OK" in r.stdout, (r.stdout[-2000:], r.stderr[-4000:])
