"""n = 4096 config-3 forward / backward under testing dispatch modes (warm,
CUDA events), with the result checked against the default mode."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1310_0956_b200 import build_geometry, build_projector  # noqa: E402


def ev(fn, reps=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
d = int(-(-n * 1.4142135623730951 // 1))
w = build_projector(build_geometry(n, d, n), precision="float32")
x = torch.rand(n * n, device="cuda")
y = torch.rand(n * d, device="cuda")
s, o = torch.empty_like(y), torch.empty_like(x)
w.forward_(x, s)
ref = s.clone()
for mode in sys.argv[2:] or ["force", "fwdskip"]:
    w.set_symmetry(mode)
    t = ev(lambda: w.forward_(x, s))
    rel = float((s - ref).norm() / ref.norm())
    print(f"n={n} {mode:10s} forward {t:7.3f} ms  rel vs default {rel:.2e}", flush=True)
