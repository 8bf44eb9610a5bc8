"""Config-3 small-grid forward (row-segment split kernels): warm CUDA-event
medians and ncu-friendly repeated launches."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1310_0956_b200 import build_geometry, build_projector  # noqa: E402

for n in (256, 512, 768):
    d = int(-(-n * 1.4142135623730951 // 1))
    w = build_projector(build_geometry(n, d, n), precision="float32")
    g = torch.Generator(device="cuda").manual_seed(3000)
    x = torch.rand(n * n, device="cuda", generator=g)
    s = torch.empty(n * d, device="cuda")
    for _ in range(5):
        w.forward_(x, s)
    torch.cuda.synchronize()
    ts = []
    for _ in range(30):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        w.forward_(x, s)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    print(f"n={n}: forward median {ts[15]:.1f} us best {ts[0]:.1f}", flush=True)
