"""Config-1 CGLS (fast fp64 pair, graph-captured iterations): a short solve
for an ncu launch list (where a CGLS iteration's ~110 us go)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1310_0956_b200 import SolverConfig, build_geometry, build_projector, cgls_solve  # noqa

n, d, m = 256, 363, 180
g = build_geometry(n, d, m)
w = build_projector(g, precision="float64", mode="fast")
b = torch.from_numpy(np.random.default_rng(0).random(m * d)).cuda()
for its in (3, 10):
    x, rec = cgls_solve(w, b, cfg=SolverConfig(max_iterations=its, residual_tolerance=0.0))
torch.cuda.synchronize()
print("ok", len(rec.rel_residual))
