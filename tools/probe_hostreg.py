"""cudaHostRegister of a numpy array per call vs the staged copy: cost of
register + DMA + unregister for 64 / 95 MB (n = 4096 image / sinogram)."""
import time

import numpy as np
import torch

cr = torch.cuda.cudart()
for mb in (64, 95):
    a = np.random.default_rng(0).random(mb * 262144, dtype=np.float32)
    dev = torch.empty(a.size, device="cuda")
    torch.cuda.synchronize()
    for rep in range(4):
        t0 = time.perf_counter()
        ptr = a.ctypes.data
        rc = cr.cudaHostRegister(ptr, a.nbytes, 0)
        t1 = time.perf_counter()
        dev.copy_(torch.from_numpy(a), non_blocking=True)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        rc2 = cr.cudaHostUnregister(ptr)
        t3 = time.perf_counter()
        print(f"{mb} MB rc {rc} {rc2}: register {1e3*(t1-t0):.2f} ms  copy {1e3*(t2-t1):.2f} ms "
              f"({a.nbytes/(t2-t1)/1e9:.1f} GB/s)  unregister {1e3*(t3-t2):.2f} ms", flush=True)
    # fresh array each time (a solver's new vector): pages not yet touched by the driver
    for rep in range(3):
        b = a.copy()
        t0 = time.perf_counter()
        cr.cudaHostRegister(b.ctypes.data, b.nbytes, 0)
        t1 = time.perf_counter()
        dev.copy_(torch.from_numpy(b), non_blocking=True)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        cr.cudaHostUnregister(b.ctypes.data)
        t3 = time.perf_counter()
        print(f"{mb} MB fresh: register {1e3*(t1-t0):.2f} copy {1e3*(t2-t1):.2f} unregister {1e3*(t3-t2):.2f}", flush=True)
