"""Host<->device copy paths for the numpy drop-in call (64 MB image, 95 MB
sinogram, float32): pageable .to()/.cpu() vs staging through pinned memory."""
import time

import numpy as np
import torch

dev = torch.device("cuda", 0)
for nbytes in (64 << 20, 95 << 20):
    a = np.random.default_rng(0).uniform(0, 1, nbytes // 4).astype(np.float32)
    d = torch.empty(a.size, dtype=torch.float32, device=dev)
    def t(fn, reps=10):
        fn(); torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / reps
    pin = torch.empty(a.size, dtype=torch.float32).pin_memory()
    pn = pin.numpy()
    res = {}
    res["h2d_pageable"] = t(lambda: d.copy_(torch.from_numpy(a)))
    res["h2d_pinned_only"] = t(lambda: d.copy_(pin, non_blocking=True))
    res["h2d_copyto_pinned"] = t(lambda: (np.copyto(pn, a), d.copy_(pin, non_blocking=True)))
    res["d2h_cpu"] = t(lambda: d.cpu())
    res["d2h_pinned_only"] = t(lambda: pin.copy_(d, non_blocking=True))
    def d2h_new_pinned():
        h = torch.empty(a.size, dtype=torch.float32, pin_memory=True)
        h.copy_(d, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return h.numpy()
    res["d2h_cached_pinned"] = t(d2h_new_pinned)
    print(nbytes >> 20, "MB", {k: f"{nbytes / v / 1e9:.1f} GB/s ({v*1e3:.2f} ms)" for k, v in res.items()})
