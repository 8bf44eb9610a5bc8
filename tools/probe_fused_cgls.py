"""Config-1 CGLS / WMG-CGLS to 1e-4 with the fused CGLS kernels on and off
(best of 5, synchronised wall clock, graphs cached)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1310_0956_b200 import (SolverConfig, build_geometry, build_projector,  # noqa: E402
                                  build_wmg_hierarchy, cgls_solve, random_ellipses,
                                  wmg_preconditioner)
from paper_1310_0956_b200 import solvers as S  # noqa: E402

n, d, m = 256, 363, 180
w = build_projector(build_geometry(n, d, m), precision="float64", mode="fast")
x_ex = random_ellipses(n, 20, seed=1000)
b = w @ x_ex
b = b + 0.01 * np.abs(b).max() * np.random.default_rng(1500).standard_normal(b.size)
bd = torch.from_numpy(b).cuda()
cfg = SolverConfig(max_iterations=400, residual_tolerance=1e-4)


def best(fn, reps=5):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return min(ts), out


for fused in (True, False, True, False):
    S.FUSED_CGLS = fused
    cgls_solve(w, bd, cfg=cfg)
    t, (_, rec) = best(lambda: cgls_solve(w, bd, cfg=cfg))
    line = f"fused={fused}: CGLS {t * 1e3:.2f} ms ({rec.iterations[-1]} its)"
    for nu in (0, 2):
        h = build_wmg_hierarchy(w, n, 0.0, 3, nu_pre=nu, nu_post=nu)
        pre = wmg_preconditioner(h)
        cgls_solve(w, bd, precond=pre, cfg=cfg)
        t, (_, rec) = best(lambda: cgls_solve(w, bd, precond=pre, cfg=cfg))
        line += f"  WMG nu={nu} {t * 1e3:.2f} ms ({rec.iterations[-1]} its)"
    print(line, flush=True)
