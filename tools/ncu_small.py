"""Small-grid pairs for ncu captures: config-3 n = 512 (fp32) and config 1
(n = 256, fp64 fast), a few launches each after a warm-up."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1310_0956_b200 import build_geometry, build_projector  # noqa: E402

for (n, d, m, prec) in ((512, 725, 512, "float32"), (256, 363, 180, "float64")):
    w = build_projector(build_geometry(n, d, m), precision=prec, mode="fast")
    dt = torch.float64 if prec == "float64" else torch.float32
    x = torch.rand(n * n, dtype=dt, device="cuda")
    y = torch.rand(m * d, dtype=dt, device="cuda")
    s, o = torch.empty_like(y), torch.empty_like(x)
    for _ in range(4):
        w.forward_(x, s)
        w.backward_(y, o)
torch.cuda.synchronize()
print("ok")
