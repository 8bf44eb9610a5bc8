"""Where the numpy drop-in call's time goes at n = 4096 (w @ x, w.T @ y with
float32 numpy vectors): staged H2D, kernel, D2H into pinned pool buffers."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1310_0956_b200 import _device as D  # noqa: E402
from paper_1310_0956_b200 import build_geometry, build_projector  # noqa: E402

n = 4096
d = int(-(-n * 1.4142135623730951 // 1))
w = build_projector(build_geometry(n, d, n), precision="float32")
rng = np.random.default_rng(0)
x = rng.random(n * n, dtype=np.float32)
y = rng.random(n * d, dtype=np.float32)
for th in [int(a) for a in sys.argv[1:]] or [4]:
    D._STAGE_THREADS = th
    for _ in range(3):
        s = w @ x
        i = w.T @ y
    torch.cuda.synchronize()
    T = {"h2d_x": 0, "fwd": 0, "d2h_s": 0, "h2d_y": 0, "bwd": 0, "d2h_i": 0, "pair": 0}
    R = 5
    for _ in range(R):
        t0 = time.perf_counter()
        xd, _ = D.to_device(x, torch.float32)
        torch.cuda.synchronize(); t1 = time.perf_counter()
        sd = torch.empty(w.shape[0], device="cuda")
        w.forward_(xd, sd)
        torch.cuda.synchronize(); t2 = time.perf_counter()
        s = D.to_caller(sd, True)
        t3 = time.perf_counter()
        yd, _ = D.to_device(y, torch.float32)
        torch.cuda.synchronize(); t4 = time.perf_counter()
        idd = torch.empty(w.shape[1], device="cuda")
        w.backward_(yd, idd)
        torch.cuda.synchronize(); t5 = time.perf_counter()
        i = D.to_caller(idd, True)
        t6 = time.perf_counter()
        del s, i
        for k, v in zip(T, [t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4, t6 - t5, t6 - t0]):
            T[k] += v / R * 1e3
        t0 = time.perf_counter()
    t0 = time.perf_counter()
    for _ in range(R):
        s = w @ x
        i = w.T @ y
    torch.cuda.synchronize()
    T["dropin_pair"] = (time.perf_counter() - t0) / R * 1e3
    print(f"threads {th}: " + " ".join(f"{k} {v:.2f}" for k, v in T.items()), flush=True)
