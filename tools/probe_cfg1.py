"""Probe config 1 (256^2, 180 angles, fp64): kernel and solver timings."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1310_0956_b200 import (SolverConfig, add_gaussian_noise, build_geometry,
                                  build_projector, build_wmg_hierarchy, cgls_solve,
                                  random_ellipses, wmg_preconditioner)


def timeit(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


out = {}
n, d, m = 256, 363, 180
g = build_geometry(n, d, m)
x_ex = random_ellipses(n, 20, seed=1000)
for mode in ("parity", "fast"):
    w = build_projector(g, mode=mode)
    x = torch.from_numpy(x_ex).cuda()
    y = torch.empty(w.shape[0], dtype=torch.float64, device="cuda")
    z = torch.empty(w.shape[1], dtype=torch.float64, device="cuda")
    out[f"{mode}_fwd_ms"] = timeit(lambda: w.forward_(x, y))
    out[f"{mode}_bwd_ms"] = timeit(lambda: w.backward_(y, z))
w = build_projector(g)
b0 = w @ x_ex
b = add_gaussian_noise(b0, 0.01, seed=1500)
for lam in (0.0,):
    for nu in (0, 2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        h = build_wmg_hierarchy(w, n, lam, 3, nu_pre=nu, nu_post=nu)
        torch.cuda.synchronize()
        t_setup = time.perf_counter() - t0
        M = wmg_preconditioner(h)
        r = torch.from_numpy(np.random.default_rng(0).standard_normal(n * n)).cuda()
        zz = torch.empty_like(r)
        t_v = timeit(lambda: M.apply_(r, zz), reps=5)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        xs, rec = cgls_solve(w, b, precond=M, x_ex=x_ex,
                             cfg=SolverConfig(max_iterations=100, residual_tolerance=1e-4,
                                              regularization_lambda=lam))
        torch.cuda.synchronize()
        t_solve = time.perf_counter() - t0
        out[f"wmg_lam{lam}_nu{nu}"] = {"setup_s": t_setup, "vcycle_ms": t_v, "solve_s": t_solve,
                                       "iters": rec.iterations[-1], "status": rec.status,
                                       "rel_res": rec.rel_residual[-1],
                                       "rel_err": rec.rel_err_l2[-1]}
torch.cuda.synchronize()
t0 = time.perf_counter()
xs, rec = cgls_solve(w, b, x_ex=x_ex, cfg=SolverConfig(max_iterations=500, residual_tolerance=1e-4))
torch.cuda.synchronize()
out["cgls"] = {"solve_s": time.perf_counter() - t0, "iters": rec.iterations[-1],
               "status": rec.status, "rel_err": rec.rel_err_l2[-1]}
print(json.dumps(out, indent=1))
