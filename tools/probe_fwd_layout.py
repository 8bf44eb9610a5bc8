"""A/B: symmetric forward block layouts (4 adjacent angles x 32 rays vs 128 rays)."""
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
    w = build_projector(build_geometry(n, d, n), precision="float32")
    x = torch.rand(n * n, device="cuda")
    s1 = torch.empty(n * d, device="cuda")
    s2 = torch.empty(n * d, device="cuda")
    w.set_symmetry("force")
    t4 = ev_time(lambda: w.forward_(x, s1))
    w.set_symmetry("fwd1")
    t1 = ev_time(lambda: w.forward_(x, s2))
    s3 = torch.empty(n * d, device="cuda")
    w.set_symmetry("lockstep")
    tl = ev_time(lambda: w.forward_(x, s3))
    s4 = torch.empty(n * d, device="cuda")
    w.set_symmetry("fwdrows")
    tm = ev_time(lambda: w.forward_(x, s4))
    s5 = torch.empty(n * d, device="cuda")
    w.set_symmetry("plainplanes")
    tp = ev_time(lambda: w.forward_(x, s5))
    torch.cuda.synchronize()
    torch.cuda.synchronize()
    out[n] = {"fwd_default_ms": t4, "fwd_1angle_ms": t1, "fwd_lockstep_ms": tl, "fwd_rows_ms": tm, "fwd_plainplanes_ms": tp,
              "plain_max_rel_diff": float((s1 - s5).abs().max() / s1.abs().max()),
              "rows_max_rel_diff": float((s1 - s4).abs().max() / s1.abs().max()),
              "max_abs_diff": float((s1 - s2).abs().max()),
              "lockstep_max_rel_diff": float((s1 - s3).abs().max() / s1.abs().max())}
print(json.dumps(out, indent=1))
