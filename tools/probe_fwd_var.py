"""Symmetric-forward block shapes (WMG_FWD_VAR, read once per process): time
the n-grid forward warm with CUDA events and compare the sinogram with the
default shape's (saved by the VAR=0 run)."""
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_1310_0956_b200 import build_geometry, build_projector  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
d = int(-(-n * 1.4142135623730951 // 1))
w = build_projector(build_geometry(n, d, n), precision="float32")
g = torch.Generator(device="cuda").manual_seed(3000)
x = torch.rand(n * n, device="cuda", generator=g)
s = torch.empty(n * d, device="cuda")
for _ in range(3):
    w.forward_(x, s)
torch.cuda.synchronize()
ts = []
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    w.forward_(x, s)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
var = os.environ.get("WMG_FWD_VAR", "0")
path = f"/tmp/fwd_ref_{n}.pt"
if var == "0":
    torch.save(s.cpu(), path)
    rel = 0.0
else:
    ref = torch.load(path).cuda()
    rel = float((s - ref).norm() / ref.norm())
print(f"n={n} var={var} forward median {ts[5]:.3f} best {ts[0]:.3f} ms rel {rel:.1e}", flush=True)
