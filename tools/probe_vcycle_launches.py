"""One config-1 V-cycle (nu = 2+2), eager, between cudaProfilerStart/Stop."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1310_0956_b200 import (build_geometry, build_projector, build_wmg_hierarchy,  # noqa
                                  wmg_preconditioner)

n, d, m = 256, 363, 180
w = build_projector(build_geometry(n, d, m))
h = build_wmg_hierarchy(w, n, 0.0, 3, nu_pre=2, nu_post=2)
M = wmg_preconditioner(h, graph=False)
v = torch.randn(n * n, dtype=torch.float64, device="cuda")
o = torch.empty_like(v)
M.apply_(v, o)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
M.apply_(v, o)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok")
