"""Config-4 geometry (n = 2048, 1024 angles, 2897 detectors) fp32 pair: the default
forward dispatch (8-segment form, < 8000 blocks) against the unsplit form
(set_symmetry("fwdflat")), alone and with two solves' pairs on two streams."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1310_0956_b200 import build_geometry, build_projector  # noqa: E402

n, d, m = 2048, 2897, 1024
g = build_geometry(n, d, m)
for mode in (True, "fwdflat"):
    ws = [build_projector(g, precision="float32") for _ in range(2)]
    for w in ws:
        w.set_symmetry(mode)
    xs = [torch.rand(n * n, device="cuda") for _ in range(2)]
    ys = [torch.rand(m * d, device="cuda") for _ in range(2)]
    ss = [torch.empty(m * d, device="cuda") for _ in range(2)]
    os_ = [torch.empty(n * n, device="cuda") for _ in range(2)]
    streams = [torch.cuda.Stream() for _ in range(2)]

    def pair(i):
        ws[i].forward_(xs[i], ss[i])
        ws[i].backward_(ys[i], os_[i])

    for _ in range(3):
        pair(0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(50):
        pair(0)
    torch.cuda.synchronize()
    t1 = (time.perf_counter() - t0) / 50
    for _ in range(3):
        for i in range(2):
            with torch.cuda.stream(streams[i]):
                pair(i)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(50):
        for i in range(2):
            with torch.cuda.stream(streams[i]):
                pair(i)
    torch.cuda.synchronize()
    t2 = (time.perf_counter() - t0) / 50
    print(f"mode={mode}: one stream {t1 * 1e3:.3f} ms per pair; two streams {t2 * 1e3:.3f} ms per "
          f"two pairs ({t2 * 5e2:.3f} per pair)", flush=True)
