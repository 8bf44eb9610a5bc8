"""Profile one cached-graph WMG-CGLS solve (config 1, nu = 2) between
cudaProfilerStart/Stop: run under ncu --profile-from-start off."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1310_0956_b200 import (SolverConfig, add_gaussian_noise, build_geometry,  # noqa: E402
                                  build_projector, build_wmg_hierarchy, cgls_solve,
                                  random_ellipses, wmg_preconditioner)

mode = sys.argv[1] if len(sys.argv) > 1 else "fast"
n, d, m = 256, 363, 180
g = build_geometry(n, d, m)
w = build_projector(g)
wf = build_projector(g, precision="float64", mode="fast")
x_ex = random_ellipses(n, 20, seed=1000)
b = add_gaussian_noise(w @ x_ex, 0.01, seed=1500)
bd = torch.from_numpy(b).cuda()
h = build_wmg_hierarchy(w, n, 0.0, 3, nu_pre=2, nu_post=2, node_mode=mode)
M = wmg_preconditioner(h)
cfg = SolverConfig(max_iterations=3, residual_tolerance=1e-4)
cgls_solve(wf, bd, precond=M, cfg=cfg)
cgls_solve(wf, bd, precond=M, cfg=cfg)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
cgls_solve(wf, bd, precond=M, cfg=SolverConfig(max_iterations=2, residual_tolerance=1e-4))
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("done")
