"""Small-grid (config 1, 256^2 / 180 x 363) projector timings per kernel path."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1310_0956_b200 import build_geometry, build_projector  # noqa: E402


def ev_time(fn, reps=50):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3   # us


out = {}
for (n, d, m) in ((256, 363, 180), (1024, 1449, 720)):
    g = build_geometry(n, d, m)
    for prec, dt in (("float64", torch.float64), ("float32", torch.float32)):
        for sym in (True, "force", False):
            w = build_projector(g, precision=prec, mode="fast")
            w.set_symmetry(sym)
            x = torch.rand(n * n, dtype=dt, device="cuda")
            y = torch.rand(m * d, dtype=dt, device="cuda")
            o = torch.empty_like(x)
            s = torch.empty_like(y)
            out[f"n{n}_{prec}_sym{sym}"] = {
                "fwd_us": ev_time(lambda: w.forward_(x, s)),
                "bwd_us": ev_time(lambda: w.backward_(y, o))}
print(json.dumps(out, indent=1))
