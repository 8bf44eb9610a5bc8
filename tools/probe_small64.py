"""Small-grid float64 backprojector A/B (WMG_SMALL64 read once per process):
warm CUDA-event times of the single and sibling-batched (B = 3) launches, and
the result against the float64 parity backprojector (reference W^T y)."""
import os
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


tag = "small64"
for n, d, m in ((256, 363, 180), (128, 182, 90), (512, 725, 360), (64, 91, 90), (256, 363, 64)):
    g = build_geometry(n, d, m)
    w = build_projector(g, precision="float64", mode="fast")
    wp = build_projector(g)
    gen = torch.Generator(device="cuda").manual_seed(1)
    y = torch.rand(m * d, dtype=torch.float64, device="cuda", generator=gen)
    S3 = torch.rand(3, m * d, dtype=torch.float64, device="cuda", generator=gen)
    o = torch.empty(n * n, dtype=torch.float64, device="cuda")
    O3 = torch.empty(3, n * n, dtype=torch.float64, device="cuda")
    tb = ev(lambda: w.backward_(y, o))
    tb3 = ev(lambda: w.backward_batch_(S3, O3))
    ref = wp.backward(y)
    rel = float((o - ref).norm() / ref.norm())
    ref3 = torch.stack([wp.backward(S3[i]) for i in range(3)])
    rel3 = float((O3 - ref3).norm() / ref3.norm())
    same = all(torch.equal(O3[i], w.backward(S3[i])) for i in range(3))
    print(f"{tag} n={n} m={m}: backward {tb:6.1f} us  B3 {tb3:6.1f} us  rel vs parity {rel:.1e} "
          f"/ {rel3:.1e}  batch==single {same}", flush=True)
