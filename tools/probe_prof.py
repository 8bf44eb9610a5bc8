import sys, time
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
cfg = SolverConfig(max_iterations=100, residual_tolerance=1e-4)
for _ in range(2):
    cgls_solve(wf, b, precond=M, cfg=cfg)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    cgls_solve(wf, b, precond=M, cfg=cfg)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=25))
t0 = time.perf_counter(); cgls_solve(wf, b, precond=M, cfg=cfg); torch.cuda.synchronize(); print("solve", time.perf_counter() - t0)
import cProfile, pstats
pr = cProfile.Profile(); pr.enable(); cgls_solve(wf, b, precond=M, cfg=cfg); torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
