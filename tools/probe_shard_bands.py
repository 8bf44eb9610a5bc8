"""Cost of running a rank's backprojection in the 4 band groups the allreduce
overlap uses (AngleShardedProjector._band_groups) against one launch, for
rank 0's quad shard at n = 4096 (one GPU, no collective)."""
import math
import sys

import torch

sys.path.insert(0, ".")
from paper_1310_0956_b200 import build_geometry, build_projector  # noqa: E402
from paper_1310_0956_b200.sharding import AngleShardedProjector, shard_angles  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
d = int(math.ceil(n * math.sqrt(2.0)))
g = build_geometry(n, d, n)
for world in (1, 2, 4, 8):
    idx = shard_angles(n, world, 0, "quad")
    w = build_projector(g.subset(idx), precision="float32")
    y = torch.rand(len(idx) * d, device="cuda")
    o = torch.empty(n * n, device="cuda")
    qt = w.backward_bands()
    line = [f"world={world}"]
    for groups in (1, 2, 4):
        helper = AngleShardedProjector.__new__(AngleShardedProjector)
        helper.overlap_groups = groups
        bands = helper._band_groups(qt)

        def run():
            for s0, s1 in bands:
                w.backward_band_(y, o, s0, s1)
        for _ in range(3):
            run()
        ts = []
        for _ in range(7):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            run()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        line.append(f"{groups} groups {ts[3]:.3f} ms")
    print("  ".join(line), flush=True)
