"""fp64 fast symmetric forward: mixed warps (default) vs one angle per block."""
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
for n, d, m in ((1024, 1449, 720), (2048, 2897, 1024)):
    w = build_projector(build_geometry(n, d, m), precision="float64", mode="fast")
    x = torch.rand(n * n, dtype=torch.float64, device="cuda")
    s1 = torch.empty(m * d, dtype=torch.float64, device="cuda")
    s2 = torch.empty(m * d, dtype=torch.float64, device="cuda")
    w.set_symmetry(True)
    t1 = ev_time(lambda: w.forward_(x, s1))
    w.set_symmetry("fwdrows")
    t2 = ev_time(lambda: w.forward_(x, s2))
    torch.cuda.synchronize()
    out[n] = {"mix_ms": t1, "rows_ms": t2,
              "max_rel_diff": float((s1 - s2).abs().max() / s2.abs().max())}
print(json.dumps(out, indent=1))
