"""to_caller (pinned pool) vs a manual pinned copy, 64 / 95 MB float32."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1310_0956_b200 import _device as D  # noqa: E402

for nb in (64 << 20, 95 << 20):
    d = torch.rand(nb // 4, device="cuda")
    torch.cuda.synchronize()
    for rep in range(3):
        ts = []
        for _ in range(6):
            t0 = time.perf_counter()
            a = D.to_caller(d, True)
            ts.append(time.perf_counter() - t0)
            del a
        pin = torch.empty(nb // 4, pin_memory=True)
        t0 = time.perf_counter()
        pin.copy_(d, non_blocking=True)
        torch.cuda.synchronize()
        tm = time.perf_counter() - t0
        print(nb >> 20, "MB to_caller ms:", " ".join(f"{1e3 * x:.2f}" for x in ts),
              f"| manual pinned {1e3 * tm:.2f}", flush=True)
