"""Config-1 WMG-CGLS with float64 vs float32 node projectors (node_mode)."""
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
for mode in ("fast", "fast32", "fast", "fast32"):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    M = wmg_preconditioner(build_wmg_hierarchy(w, n, 0.0, 3, nu_pre=2, nu_post=2,
                                               node_mode=mode))
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    _, rec = cgls_solve(wf, bd, precond=M, cfg=cfg)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    v = torch.randn(n * n, dtype=torch.float64, device="cuda")
    o = torch.empty_like(v)
    M.apply_(v, o)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    for _ in range(20):
        M.apply_(v, o)
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    print(f"{mode}: setup {t1-t0:.4f} s  solve {t2-t1:.4f} s  its {rec.iterations[-1]} "
          f"rel {rec.rel_residual[-1]:.3e}  V-cycle {(t4-t3)/20*1e3:.3f} ms", flush=True)
