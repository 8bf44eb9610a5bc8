"""A/B: symmetric backprojector warp layouts (2-D 8x4 blocks vs lane = column)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1310_0956_b200 import build_geometry, build_projector  # noqa: E402


def ev_time(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


out = {}
for n in (1024, 2048, 4096):
    d = int(-(-n * 2 ** 0.5 // 1))
    g = build_geometry(n, d, n)
    w = build_projector(g, precision="float32")
    y = torch.rand(n * d, device="cuda")
    o1 = torch.empty(n * n, device="cuda")
    o2 = torch.empty(n * n, device="cuda")
    w.set_symmetry("force")
    t2d = ev_time(lambda: w.backward_(y, o1))
    w.backward_(y, o1)
    w.set_symmetry("rowlayout")
    trow = ev_time(lambda: w.backward_(y, o2))
    w.backward_(y, o2)
    torch.cuda.synchronize()
    rel = ((o1 - o2).abs().max() / o2.abs().max()).item()
    out[n] = {"bwd_2d_ms": t2d, "bwd_row_ms": trow, "max_rel_diff": rel}
print(json.dumps(out, indent=1))
