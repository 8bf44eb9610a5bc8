"""Per-rank efficiency of the angle-sharded pair at n = 4096: forward / backward of
rank 0's quad shard for world = 1, 2, 4, 8 (one GPU, no collective) against
1 / world of the unsharded time."""
import math
import sys

import torch

sys.path.insert(0, ".")
from paper_1310_0956_b200 import build_geometry, build_projector  # noqa: E402
from paper_1310_0956_b200.sharding import shard_angles  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
d = int(math.ceil(n * math.sqrt(2.0)))
g = build_geometry(n, d, n)
x = torch.rand(n * n, device="cuda")
base = None
for world in (1, 2, 4, 8):
    idx = shard_angles(n, world, 0, "quad")
    w = build_projector(g.subset(idx), precision="float32")
    m = len(idx)
    y = torch.rand(m * d, device="cuda")
    s, o = torch.empty_like(y), torch.empty_like(x)
    for _ in range(3):
        w.forward_(x, s)
        w.backward_(y, o)
    res = []
    for fn in (lambda: w.forward_(x, s), lambda: w.backward_(y, o)):
        ts = []
        for _ in range(7):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        res.append(ts[3])
    if base is None:
        base = res
    print(f"world={world} m/rank={m}: fwd {res[0]:.3f} ms (eff {base[0] / world / res[0]:.2f})  "
          f"bwd {res[1]:.3f} ms (eff {base[1] / world / res[1]:.2f})  bands={w.backward_bands()}",
          flush=True)
    del w
