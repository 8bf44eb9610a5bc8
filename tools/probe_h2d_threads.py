"""wmg_h2d_staged: host threads x chunk size sweep for the 64 MB image and the
95 MB sinogram of the n = 4096 numpy drop-in call (warm, 10 reps, synchronised)."""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1310_0956_b200 import _native as N  # noqa: E402

dev = torch.device("cuda", 0)
torch.cuda.set_device(0)
st = torch.cuda.current_stream(dev)
for nbytes in (64 << 20, 95 << 20):
    a = np.random.default_rng(0).uniform(0, 1, nbytes // 4).astype(np.float32)
    d = torch.empty(a.size, dtype=torch.float32, device=dev)
    pin = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    line = [f"{nbytes >> 20} MB:"]
    for thr in (2, 4, 6, 8, 10, 12, 14, 16):
        def run():
            N.call("wmg_h2d_staged", d.data_ptr(), a.ctypes.data, a.nbytes, pin.data_ptr(), thr,
                   st.cuda_stream)
            st.synchronize()
        run()
        run()
        t0 = time.perf_counter()
        for _ in range(10):
            run()
        dt = (time.perf_counter() - t0) / 10
        line.append(f"{thr}t {dt * 1e3:.2f} ms ({nbytes / dt / 1e9:.1f} GB/s)")
    print("  ".join(line), flush=True)
    # pure host memcpy and pure DMA for reference
    pn = pin.numpy().view(np.float32)
    t0 = time.perf_counter()
    for _ in range(5):
        np.copyto(pn, a)
    print(f"   single-thread np.copyto {(time.perf_counter() - t0) / 5 * 1e3:.2f} ms", end="")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        d.copy_(torch.from_numpy(pn), non_blocking=True)
        st.synchronize()
    print(f"   pinned DMA {(time.perf_counter() - t0) / 10 * 1e3:.2f} ms", flush=True)
