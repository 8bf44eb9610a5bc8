"""Warm-cache CUDA-event times of the config-1 float64 fast pair (n = 256) and of
its sibling-batched form, per forward mode ('auto' vs the plain split kernel)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1310_0956_b200 import build_geometry, build_projector  # noqa: E402


def ev(fn, reps=200):
    for _ in range(5):
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
x = torch.rand(n * n, dtype=torch.float64, device="cuda")
y = torch.rand(m * d, dtype=torch.float64, device="cuda")
s = torch.empty_like(y)
o = torch.empty_like(x)
X3 = torch.rand(3, n * n, dtype=torch.float64, device="cuda")
S3 = torch.empty(3, m * d, dtype=torch.float64, device="cuda")
ref = None
for mode in ("auto",):
    w.set_symmetry(True if mode == "auto" else mode)
    tf = ev(lambda: w.forward_(x, s))
    tb = ev(lambda: w.backward_(y, o))
    tf3 = ev(lambda: w.forward_batch_(X3, S3))
    w.forward_(x, s)
    if ref is None:
        ref = s.clone()
    rel = ((s - ref).abs().max() / ref.abs().max()).item()
    print(f"{mode:10s}: forward {tf:6.1f} us  backward {tb:6.1f} us  forward batch3 {tf3:6.1f} us"
          f"  rel {rel:.1e}", flush=True)
