"""Host staging copy rate: np.copyto vs ctypes.memmove from k Python threads
(ctypes releases the GIL) into a pinned buffer, 64 MB."""
import ctypes
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

a = np.random.default_rng(0).random(64 * 262144, dtype=np.float32)
pin = torch.empty(a.nbytes, dtype=torch.uint8).pin_memory()
hp = pin.numpy().view(np.float32)
for k in (1, 2, 4, 8, 12, 16):
    pool = ThreadPoolExecutor(k)
    b = [(i * a.size) // k for i in range(k + 1)]
    for name, fn in (("copyto", lambda i: np.copyto(hp[b[i]:b[i + 1]], a[b[i]:b[i + 1]])),
                     ("memmove", lambda i: ctypes.memmove(hp.ctypes.data + 4 * b[i],
                                                          a.ctypes.data + 4 * b[i],
                                                          4 * (b[i + 1] - b[i])))):
        best = 1e9
        for _ in range(5):
            t0 = time.perf_counter()
            list(pool.map(fn, range(k)))
            best = min(best, time.perf_counter() - t0)
        print(f"threads {k:2d} {name:8s} {best*1e3:6.2f} ms {a.nbytes/best/1e9:5.1f} GB/s", flush=True)
    pool.shutdown()
