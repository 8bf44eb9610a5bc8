"""A/B: symmetric backprojector layouts -- run layout (R = 8 / R = 4 rows per
thread, float2 windows) vs the 8x4 warp blocks with float4 windows."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1310_0956_b200 import build_geometry, build_projector  # noqa: E402


def ev_time(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


out = {}
for n in [int(a) for a in sys.argv[1:]] or (1024, 2048, 4096):
    d = int(-(-n * 2 ** 0.5 // 1))
    g = build_geometry(n, d, n)
    w = build_projector(g, precision="float32")
    y = torch.rand(n * d, device="cuda")
    res = {}
    outs = {}
    for mode in (True, "bwdrun", "bwdsym8", "bwd8x4"):
        w.set_symmetry(mode)
        o = torch.empty(n * n, device="cuda")
        res[str(mode)] = ev_time(lambda: w.backward_(y, o))
        w.backward_(y, o)
        outs[str(mode)] = o
    torch.cuda.synchronize()
    ref = outs["bwd8x4"]
    for k, o in outs.items():
        res[k + "_rel"] = ((o - ref).abs().max() / ref.abs().max()).item()
    out[n] = res
print(json.dumps(out, indent=1))
