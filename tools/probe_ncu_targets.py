"""Launch the kernels to capture with ncu --set full (one of each):
  pair at n=4096 (symmetric fwd/bwd), pair at 256^2/180x363 fp64 (split kernels),
  one sparse leaf Gram at config 2."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1310_0956_b200 import build_geometry, build_projector  # noqa: E402
from paper_1310_0956_b200.multilevel import _assemble_leaf_grams, _leaf_paths  # noqa: E402

what = sys.argv[1]
if what == "pair4096":
    n, d, m = 4096, 5793, 4096
    w = build_projector(build_geometry(n, d, m), precision="float32")
    x, y = torch.rand(n * n, device="cuda"), torch.rand(m * d, device="cuda")
    s, o = torch.empty(m * d, device="cuda"), torch.empty(n * n, device="cuda")
    w.forward_(x, s)
    w.backward_(y, o)
elif what == "small":
    n, d, m = 256, 363, 180
    w = build_projector(build_geometry(n, d, m), precision="float64", mode="fast")
    x = torch.rand(n * n, dtype=torch.float64, device="cuda")
    y = torch.rand(m * d, dtype=torch.float64, device="cuda")
    s, o = torch.empty_like(y), torch.empty_like(x)
    w.forward_(x, s)
    w.backward_(y, o)
elif what == "gram":
    n, d, m = 1024, 1449, 720
    w = build_projector(build_geometry(n, d, m))
    _assemble_leaf_grams(w, n, 0.0, 5, paths=_leaf_paths(5)[5:6], method="sparse")
torch.cuda.synchronize()
print("ok", what)
