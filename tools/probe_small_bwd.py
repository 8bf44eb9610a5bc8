"""Config-3 small-grid backprojection: warm CUDA-event medians (host-loop bound below ~40 us)."""
import sys, torch
sys.path.insert(0, ".")
from paper_1310_0956_b200 import build_geometry, build_projector
import os
for n in (256, 512, 768):
    d = int(-(-n * 1.4142135623730951 // 1))
    w = build_projector(build_geometry(n, d, n), precision="float32")
    y = torch.rand(n * d, device="cuda")
    o = torch.empty(n * n, device="cuda")
    for _ in range(5): w.backward_(y, o)
    torch.cuda.synchronize()
    ts = []
    for _ in range(30):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); w.backward_(y, o); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    print(f"n={n}: backward median {ts[15]:.1f} us", flush=True)
