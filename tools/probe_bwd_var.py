"""Backprojector variants (env knobs read once per process): warm CUDA-event
time of the n-grid backprojection, result compared with the default's."""
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_1310_0956_b200 import build_geometry, build_projector  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
tag = sys.argv[2] if len(sys.argv) > 2 else "default"
d = int(-(-n * 1.4142135623730951 // 1))
w = build_projector(build_geometry(n, d, n), precision="float32")
g = torch.Generator(device="cuda").manual_seed(3001)
y = torch.rand(n * d, device="cuda", generator=g)
x = torch.empty(n * n, device="cuda")
for _ in range(3):
    w.backward_(y, x)
torch.cuda.synchronize()
ts = []
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    w.backward_(y, x)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
path = f"/tmp/bwd_ref_{n}.pt"
if tag == "default":
    torch.save(x.cpu(), path)
    rel = 0.0
else:
    ref = torch.load(path).cuda()
    rel = float((x - ref).norm() / ref.norm())
print(f"n={n} {tag} backward median {ts[5]:.3f} best {ts[0]:.3f} ms rel {rel:.1e}", flush=True)
