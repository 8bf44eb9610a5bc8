"""A/B of the numpy drop-in pair at n = 4096 with and without the partial
launches that copy finished rows to the host while later parts compute."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1310_0956_b200.geometry as G  # noqa: E402
from paper_1310_0956_b200 import build_geometry, build_projector  # noqa: E402

n = 4096
d = int(-(-n * 1.4142135623730951 // 1))
w = build_projector(build_geometry(n, d, n), precision="float32")
rng = np.random.default_rng(0)
x = rng.random(n * n, dtype=np.float32)
y = rng.random(n * d, dtype=np.float32)
on = G._OVERLAP_MIN_BYTES
res = {"overlap": [], "plain": []}
for rep in range(6):
    for mode in ("overlap", "plain"):
        G._OVERLAP_MIN_BYTES = on if mode == "overlap" else 1 << 62
        for _ in range(2):
            s = w @ x
            i = w.T @ y
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5):
            s = w @ x
            i = w.T @ y
        res[mode].append((time.perf_counter() - t0) / 5 * 1e3)
for k, v in res.items():
    v.sort()
    print(f"{k:8s} pair median {v[len(v) // 2]:.2f} best {v[0]:.2f} ms", flush=True)
