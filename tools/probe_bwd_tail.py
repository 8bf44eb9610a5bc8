"""Does the n = 4096 eight-image backprojector pay for its partial last wave?
2080 equal tile-pair blocks on 148 x 4 slots = 3.51 waves.  Times the banded
launch on the first B tile pairs for several B (wmg_backward_band)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1310_0956_b200 import build_geometry, build_projector  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
d = int(-(-n * 1.4142135623730951 // 1))
w = build_projector(build_geometry(n, d, n), precision="float32")
y = torch.rand(n * d, device="cuda")
o = torch.empty(n * n, device="cuda")
qt = w.backward_bands()
off = lambda s: s * qt - s * (s - 1) // 2  # noqa: E731
for _ in range(3):
    w.backward_(y, o)
for s1 in sorted(set([qt // 4, qt // 2, 34, 37, 40, 46, 52, 58, qt])):
    if s1 > qt:
        continue
    ts = []
    for _ in range(7):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        w.backward_band_(y, o, 0, s1)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    b = off(s1)
    print(f"bands [0,{s1}): {b} blocks = {b / 592:.2f} waves  {ts[3]:.3f} ms  "
          f"{ts[3] / b * 1e3:.3f} us/block", flush=True)
