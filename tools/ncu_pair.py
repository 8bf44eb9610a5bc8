"""The config-3 pair at n (default 4096) for ncu: two forward + two backward
launches of the default dispatch (fwd_sym_kernel, bwd_sym8_kernel)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1310_0956_b200 import build_geometry, build_projector  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
d = int(-(-n * 1.4142135623730951 // 1))
w = build_projector(build_geometry(n, d, n), precision="float32")
x = torch.rand(n * n, device="cuda")
y = torch.rand(n * d, device="cuda")
s, o = torch.empty_like(y), torch.empty_like(x)
for _ in range(2):
    w.forward_(x, s)
    w.backward_(y, o)
torch.cuda.synchronize()
print("ok")
