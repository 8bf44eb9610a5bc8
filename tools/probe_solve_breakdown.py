"""Config-1 WMG-CGLS: first solve (captures the CGLS iteration graph) vs repeat
solves with the same preconditioner; V-cycle replay time."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1310_0956_b200 import (SolverConfig, add_gaussian_noise, build_geometry,  # noqa
                                  build_projector, build_wmg_hierarchy, cgls_solve,
                                  random_ellipses, wmg_preconditioner)

n, d, m = 256, 363, 180
g = build_geometry(n, d, m)
w = build_projector(g)
wf = build_projector(g, precision="float64", mode="fast")
x_ex = random_ellipses(n, 20, seed=1000)
b = add_gaussian_noise(w @ x_ex, 0.01, seed=1500)
bd = torch.from_numpy(b).cuda()
cfg = SolverConfig(max_iterations=100, residual_tolerance=1e-4)
for nu in (2, 0):
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        M = wmg_preconditioner(build_wmg_hierarchy(w, n, 0.0, 3, nu_pre=nu, nu_post=nu))
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        times = []
        for k in range(3):
            _, rec = cgls_solve(wf, bd, precond=M, cfg=cfg)
            torch.cuda.synchronize()
            times.append(time.perf_counter() - t1)
            t1 = time.perf_counter()
        print(f"nu={nu} rep={rep}: setup {t1 - t0 - sum(times):.4f}s solves "
              + " ".join(f"{x*1e3:.1f}ms" for x in times) + f" its {rec.iterations[-1]}", flush=True)
