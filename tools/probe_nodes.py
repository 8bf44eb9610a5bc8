import json, sys, time
import numpy as np, torch
sys.path.insert(0, ".")
from paper_1310_0956_b200 import (SolverConfig, add_gaussian_noise, build_geometry, build_projector,
                                  build_wmg_hierarchy, cgls_solve, random_ellipses, wmg_preconditioner)
n, d, m = 256, 363, 180
g = build_geometry(n, d, m)
w = build_projector(g); wf = build_projector(g, mode="fast")
x_ex = random_ellipses(n, 20, seed=1000)
b = torch.from_numpy(add_gaussian_noise(w @ x_ex, 0.01, seed=1500)).cuda()
out = {}
for nu in (0, 2):
    for nm in ("fast", "fast32"):
        h = build_wmg_hierarchy(w, n, 0.0, 3, nu_pre=nu, nu_post=nu, node_mode=nm)
        M = wmg_preconditioner(h)
        cfg = SolverConfig(max_iterations=100, residual_tolerance=1e-4)
        cgls_solve(wf, b, precond=M, cfg=cfg)
        ts = []
        for _ in range(3):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            _, rec = cgls_solve(wf, b, precond=M, cfg=cfg)
            torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
        v = torch.randn(n * n, dtype=torch.float64, device="cuda"); o = torch.empty_like(v)
        torch.cuda.synchronize(); t0 = time.perf_counter()
        for _ in range(20): M.apply_(v, o)
        torch.cuda.synchronize()
        out[f"nu{nu}_{nm}"] = {"solve_s": min(ts), "iters": rec.iterations[-1], "status": rec.status,
                               "vcycle_ms": (time.perf_counter() - t0) / 20 * 1e3}
print(json.dumps(out, indent=1))
