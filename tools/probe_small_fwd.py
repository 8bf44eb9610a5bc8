"""Config-3 small grids: the symmetric forward's row-segment split (WMG_SEG,
read once per process) -- warm CUDA-event medians, result vs the default."""
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_1310_0956_b200 import build_geometry, build_projector  # noqa: E402

tag = os.environ.get("WMG_SEG", "default")
for n in (256, 512, 768, 1024):
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
    path = f"/tmp/sfwd_{n}.pt"
    if tag == "default":
        torch.save(s.cpu(), path)
        rel = 0.0
    else:
        ref = torch.load(path).cuda()
        rel = float((s - ref).norm() / ref.norm())
    print(f"seg={tag} n={n}: forward median {ts[15]:.1f} us best {ts[0]:.1f} rel {rel:.1e}",
          flush=True)
