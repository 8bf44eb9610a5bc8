"""Pageable H2D from several host threads at once (each thread one chunk on its
own stream, the driver staging internally) vs the native staged copy."""
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1310_0956_b200 import _device as D  # noqa: E402

a = np.random.default_rng(0).random(16 << 20, dtype=np.float32)   # 64 MB
dev = torch.empty(a.size, device="cuda")
torch.cuda.synchronize()
for k in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(k)]
    b = [(i * a.size) // k for i in range(k + 1)]
    src = torch.from_numpy(a)

    def work(i):
        with torch.cuda.stream(streams[i]):
            dev[b[i]:b[i + 1]].copy_(src[b[i]:b[i + 1]], non_blocking=False)

    best = 1e9
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        th = [threading.Thread(target=work, args=(i,)) for i in range(k)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    print(f"pageable, {k} threads: {best * 1e3:.2f} ms ({a.nbytes / best / 1e9:.1f} GB/s)", flush=True)
for _ in range(3):
    D.to_device(a, torch.float32)
torch.cuda.synchronize()
best = 1e9
for _ in range(5):
    t0 = time.perf_counter()
    out, _ = D.to_device(a, torch.float32)
    torch.cuda.synchronize()
    best = min(best, time.perf_counter() - t0)
print(f"staged (wmg_h2d_staged): {best * 1e3:.2f} ms ({a.nbytes / best / 1e9:.1f} GB/s)")
