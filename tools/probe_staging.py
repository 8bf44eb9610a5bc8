"""H2D rate of the numpy staging path (paper_1310_0956_b200._device) vs its
host-thread count, and the pinned D2H path, for 64 / 95 MB float32 vectors."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1310_0956_b200 import _device as D  # noqa: E402

dev = torch.device("cuda", 0)
for nbytes in (64 << 20, 95 << 20):
    a = np.random.default_rng(0).uniform(0, 1, nbytes // 4).astype(np.float32)
    for th in (1, 2, 4, 8, 12):
        D._STAGE_THREADS = th
        D._pool = None
        D._stage.clear()
        for _ in range(3):
            t, _ = D.to_device(a, torch.float32, dev)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(10):
            t, _ = D.to_device(a, torch.float32, dev)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / 10
        print(f"{nbytes >> 20} MB H2D staged, {th:2d} threads: {nbytes / dt / 1e9:5.1f} GB/s", flush=True)
    t0 = time.perf_counter()
    for _ in range(10):
        D.to_caller(t, True)
    dt = (time.perf_counter() - t0) / 10
    print(f"{nbytes >> 20} MB D2H pinned: {nbytes / dt / 1e9:5.1f} GB/s", flush=True)
