"""One launch of each symmetric-forward variant at n=4096 (for ncu metrics)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1310_0956_b200 import build_geometry, build_projector  # noqa: E402

n, d = 4096, 5793
w = build_projector(build_geometry(n, d, n), precision="float32")
x = torch.rand(n * n, device="cuda")
s = torch.empty(n * d, device="cuda")
for mode in ("force", "fwd1", "lockstep", "fwdrows"):
    w.set_symmetry(mode)
    w.forward_(x, s)
torch.cuda.synchronize()
print("ok")
