import sys
import numpy as np, torch
sys.path.insert(0, ".")
from paper_1310_0956_b200 import (SolverConfig, add_gaussian_noise, build_geometry, build_projector,
                                  build_wmg_hierarchy, cgls_solve, random_ellipses, wmg_preconditioner)
n, d, m = 256, 363, 180
g = build_geometry(n, d, m)
w = build_projector(g); wf = build_projector(g, mode="fast")
x_ex = random_ellipses(n, 20, seed=1000)
b = torch.from_numpy(add_gaussian_noise(w @ x_ex, 0.01, seed=1500)).cuda()
h = build_wmg_hierarchy(w, n, 0.0, 3)
M = wmg_preconditioner(h)
cfg = SolverConfig(max_iterations=3, residual_tolerance=1e-4)
cgls_solve(wf, b, precond=M, cfg=cfg)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
cgls_solve(wf, b, precond=M, cfg=SolverConfig(max_iterations=2))
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
