"""Times of the small-grid pair under each dispatch mode (warm, CUDA events)."""
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


import sys as _s
CASES = [(256, 363, 180, "float64"), (256, 363, 180, "float32"), (512, 725, 512, "float32"),
         (1024, 1449, 1024, "float32"), (256, 363, 256, "float32")]
for (n, d, m, prec) in CASES:
    w = build_projector(build_geometry(n, d, m), precision=prec, mode="fast")
    dt = torch.float64 if prec == "float64" else torch.float32
    x = torch.rand(n * n, dtype=dt, device="cuda")
    y = torch.rand(m * d, dtype=dt, device="cuda")
    s, o = torch.empty_like(y), torch.empty_like(x)
    for mode in (True, "force", "fwdflat", "bwdrunflat", False):
        try:
            w.set_symmetry(mode)
            print(f"n={n} {prec} {str(mode):9s}: forward {ev(lambda: w.forward_(x, s)):7.1f} us"
                  f"  backward {ev(lambda: w.backward_(y, o)):7.1f} us", flush=True)
        except Exception as exc:
            print(n, prec, mode, "error", exc)
