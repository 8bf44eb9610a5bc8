"""Warm-cache CUDA-event times of the config-1 float64 fast pair (n = 256,
180 angles, 363 detectors): single products and the sibling-batched (B = 3)
forms the V-cycle launches."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1310_0956_b200 import build_geometry, build_projector  # noqa: E402


def ev(fn, reps=200):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


n, d, m = 256, 363, 180
w = build_projector(build_geometry(n, d, m), precision="float64", mode="fast")
x = torch.rand(n * n, dtype=torch.float64, device="cuda")
y = torch.rand(m * d, dtype=torch.float64, device="cuda")
s = torch.empty_like(y)
o = torch.empty_like(x)
X3 = torch.rand(3, n * n, dtype=torch.float64, device="cuda")
S3 = torch.rand(3, m * d, dtype=torch.float64, device="cuda")
O3 = torch.empty_like(X3)
tf = ev(lambda: w.forward_(x, s))
tb = ev(lambda: w.backward_(y, o))
tf3 = ev(lambda: w.forward_batch_(X3, S3))
tb3 = ev(lambda: w.backward_batch_(S3, O3))
nnz = w.nnz()
print(f"n=256 fp64 fast: forward {tf:6.1f} us  backward {tb:6.1f} us  forward B3 {tf3:6.1f} us"
      f"  backward B3 {tb3:6.1f} us  nnz {nnz}  pair upd/s {2 * nnz / (tf + tb) * 1e6:.3e}"
      f"  (fp64 gather peak 148*16*1.965e9 = 4.65e12)", flush=True)
w32 = build_projector(build_geometry(n, d, m), precision="float32")
xf, yf = x.float(), y.float()
sf, of = s.float(), o.float()
print(f"n=256 fp32 fast: forward {ev(lambda: w32.forward_(xf, sf)):6.1f} us  backward "
      f"{ev(lambda: w32.backward_(yf, of)):6.1f} us", flush=True)
for nn in (512, 1024):
    dd = int(-(-nn * 1.4142135623730951 // 1))
    wq = build_projector(build_geometry(nn, dd, nn), precision="float32")
    xq = torch.rand(nn * nn, device="cuda")
    yq = torch.rand(nn * dd, device="cuda")
    sq = torch.empty_like(yq)
    oq = torch.empty_like(xq)
    tfq, tbq = ev(lambda: wq.forward_(xq, sq)), ev(lambda: wq.backward_(yq, oq))
    nz = wq.nnz()
    print(f"n={nn} fp32 config3: forward {tfq:7.1f} us  backward {tbq:7.1f} us  pair gather frac "
          f"{2 * nz / ((tfq + tbq) * 1e-6) / (148 * 32 * 1.965e9):.3f}", flush=True)
