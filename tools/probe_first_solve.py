"""cProfile of the first WMG-CGLS solve on a fresh preconditioner (config 1)."""
import cProfile
import pstats
import sys

import torch

sys.path.insert(0, ".")
from paper_1310_0956_b200 import (SolverConfig, add_gaussian_noise, build_geometry,  # noqa
                                  build_projector, build_wmg_hierarchy, cgls_solve,
                                  random_ellipses, wmg_preconditioner)

n, d, m = 256, 363, 180
g = build_geometry(n, d, m)
w = build_projector(g)
wf = build_projector(g, precision="float64", mode="fast")
b = add_gaussian_noise(w @ random_ellipses(n, 20, seed=1000), 0.01, seed=1500)
bd = torch.from_numpy(b).cuda()
cfg = SolverConfig(max_iterations=100, residual_tolerance=1e-4)
M = wmg_preconditioner(build_wmg_hierarchy(w, n, 0.0, 3, nu_pre=2, nu_post=2))
cgls_solve(wf, bd, precond=M, cfg=cfg)
M = wmg_preconditioner(build_wmg_hierarchy(w, n, 0.0, 3, nu_pre=2, nu_post=2))
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
cgls_solve(wf, bd, precond=M, cfg=cfg)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
