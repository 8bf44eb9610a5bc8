"""Forward of rank 0's quad shard (world from argv, n = 4096) for an ncu capture."""
import math
import sys

import torch

sys.path.insert(0, ".")
from paper_1310_0956_b200 import build_geometry, build_projector  # noqa: E402
from paper_1310_0956_b200.sharding import shard_angles  # noqa: E402

world = int(sys.argv[1]) if len(sys.argv) > 1 else 8
scheme = sys.argv[2] if len(sys.argv) > 2 else "quad"
n = 4096
d = int(math.ceil(n * math.sqrt(2.0)))
g = build_geometry(n, d, n)
w = build_projector(g.subset(shard_angles(n, world, 0, scheme)), precision="float32")
x = torch.rand(n * n, device="cuda")
s = torch.empty(w.shape[0], device="cuda")
for _ in range(2):
    w.forward_(x, s)
torch.cuda.synchronize()
print("ok", w.shape)
