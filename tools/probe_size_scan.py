"""Gather fraction of the fp32 forward / backward over grid sizes (multiples of
64; m = n angles, d = ceil(sqrt(2) n)): looks for dispatch anomalies between
the BASELINE sizes.  Warm medians, L2 flushed between launches."""
import math
import sys

import torch

sys.path.insert(0, ".")
from paper_1310_0956_b200 import build_geometry, build_projector  # noqa: E402

sizes = [int(a) for a in sys.argv[1:]] or list(range(512, 2049, 128)) + [2560, 3072, 3584]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
peak = 148 * 32 * 1.965e9
for n in sizes:
    d = int(math.ceil(n * math.sqrt(2.0)))
    w = build_projector(build_geometry(n, d, n), precision="float32")
    x = torch.rand(n * n, device="cuda")
    y = torch.rand(n * d, device="cuda")
    s, o = torch.empty_like(y), torch.empty_like(x)
    for _ in range(3):
        w.forward_(x, s)
        w.backward_(y, o)
    nnz = 4.0 / math.pi * n * n * n
    res = []
    for fn in (lambda: w.forward_(x, s), lambda: w.backward_(y, o)):
        ts = []
        for _ in range(9):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e-3)
        ts.sort()
        res.append(ts[4])
    print(f"n={n:5d}  fwd {res[0] * 1e6:9.1f} us frac {nnz / res[0] / peak:.3f}   "
          f"bwd {res[1] * 1e6:9.1f} us frac {nnz / res[1] / peak:.3f}", flush=True)
    del w
