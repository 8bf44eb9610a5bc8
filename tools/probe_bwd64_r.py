"""Small-grid float64 symmetric backprojector (config 1: n = 256, 180 angles),
rows per thread via WMG_R2 (read once per process): warm CUDA-event times of
the single and sibling-batched (B = 3) launches, result saved / compared."""
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


tag = "r2" if os.environ.get("WMG_R2") else "r4"
for n, d, m in ((256, 363, 180), (128, 182, 90), (512, 725, 360)):
    w = build_projector(build_geometry(n, d, m), precision="float64", mode="fast")
    g = torch.Generator(device="cuda").manual_seed(1)
    y = torch.rand(m * d, dtype=torch.float64, device="cuda", generator=g)
    S3 = torch.rand(3, m * d, dtype=torch.float64, device="cuda", generator=g)
    o = torch.empty(n * n, dtype=torch.float64, device="cuda")
    O3 = torch.empty(3, n * n, dtype=torch.float64, device="cuda")
    tb = ev(lambda: w.backward_(y, o))
    tb3 = ev(lambda: w.backward_batch_(S3, O3))
    path = f"/tmp/bwd64_{n}.pt"
    if tag == "r4":
        torch.save((o.cpu(), O3.cpu()), path)
        same = True
    else:
        a, b = torch.load(path)
        same = bool(torch.equal(a, o.cpu()) and torch.equal(b, O3.cpu()))
    print(f"{tag} n={n} m={m}: backward {tb:6.1f} us  B3 {tb3:6.1f} us  bitwise-same {same}",
          flush=True)
