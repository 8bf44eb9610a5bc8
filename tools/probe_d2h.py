"""Components of the D2H path of the numpy drop-in call (64 MB float32)."""
import time

import numpy as np
import torch

dev = torch.device("cuda", 0)
n = (64 << 20) // 4
d = torch.rand(n, device=dev)


def tm(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


keep = []
print("alloc pinned (fresh, freed)   %.2f ms" % (1e3 * tm(lambda: torch.empty(n, pin_memory=True))))
pin = torch.empty(n, pin_memory=True)
print("D2H into persistent pinned    %.2f ms" % (1e3 * tm(lambda: pin.copy_(d, non_blocking=True))))


def fresh():
    h = torch.empty(n, pin_memory=True)
    h.copy_(d, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return h.numpy()


print("fresh pinned + D2H + numpy    %.2f ms" % (1e3 * tm(fresh)))


def fresh_keep():
    keep.append(fresh())
    if len(keep) > 2:
        keep.pop(0)


print("same, caller keeps 2 results  %.2f ms" % (1e3 * tm(fresh_keep)))
print(".cpu().numpy()                %.2f ms" % (1e3 * tm(lambda: d.cpu().numpy())))
out = np.empty(n, dtype=np.float32)
print("D2H into np.empty (pageable)  %.2f ms" % (1e3 * tm(lambda: torch.from_numpy(out).copy_(d))))
