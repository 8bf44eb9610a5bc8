"""Where does the eight-image backprojector (bwd_sym8) start to beat the
four-image run layout?  Default dispatch vs set_symmetry("bwdsym8") / ("bwdrun")
for mid-size grids (warm, L2 flushed between launches)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1310_0956_b200 import build_geometry, build_projector  # noqa: E402

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for n in [int(a) for a in sys.argv[1:]] or (768, 1024, 1280, 1536, 1792, 1920, 2048):
    d = int(-(-n * 1.4142135623730951 // 1))
    y = torch.rand(n * d, device="cuda")
    out = {}
    ref = None
    for mode in (True, "bwdsym8", "bwdrun"):
        w = build_projector(build_geometry(n, d, n), precision="float32")
        w.set_symmetry(mode)
        o = torch.empty(n * n, device="cuda")
        for _ in range(3):
            w.backward_(y, o)
        ts = []
        for _ in range(15):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            w.backward_(y, o)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        ts.sort()
        if ref is None:
            ref = o.clone()
        rel = float((o - ref).norm() / ref.norm())
        out[str(mode)] = (ts[7], rel)
    print(f"n={n}: " + "  ".join(f"{k} {v[0]:.1f} us (rel {v[1]:.0e})" for k, v in out.items()),
          flush=True)
