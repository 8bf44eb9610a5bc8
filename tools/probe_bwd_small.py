"""fp64 backprojector timings at config 1 (256^2, 180 x 363), single and batch 3."""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_1310_0956_b200 import build_geometry, build_projector  # noqa: E402


def ev_time(fn, reps=100):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


n, d, m = 256, 363, 180
w = build_projector(build_geometry(n, d, m), precision="float64", mode="fast")
y = torch.rand(3, m * d, dtype=torch.float64, device="cuda")
x = torch.rand(3, n * n, dtype=torch.float64, device="cuda")
o = torch.empty_like(x)
s = torch.empty_like(y)
out = {"nsplit": os.environ.get("WMG_SYM64_NSPLIT", "auto"),
       "bwd1_us": ev_time(lambda: w.backward_(y[0], o[0])),
       "bwd3_us": ev_time(lambda: w.backward_batch_(y, o)),
       "fwd1_us": ev_time(lambda: w.forward_(x[0], s[0])),
       "fwd3_us": ev_time(lambda: w.forward_batch_(x, s))}
print(json.dumps(out))
