"""Break down one config-1 V-cycle (3 levels) on the GPU."""
import json, sys, time
import numpy as np, torch
sys.path.insert(0, ".")
from paper_1310_0956_b200 import build_geometry, build_projector, build_wmg_hierarchy
from paper_1310_0956_b200.sparse_kernels import cholesky_solve
from paper_1310_0956_b200.multilevel import restrict, prolong

def timeit(fn, reps=20):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

n, d, m = 256, 363, 180
g = build_geometry(n, d, m)
w = build_projector(g)
h = build_wmg_hierarchy(w, n, 0.0, 3)
out = {}
root = h.root
v = torch.randn(n * n, dtype=torch.float64, device="cuda")
o = torch.empty_like(v)
out["root_apply_ms"] = timeit(lambda: root.apply_system_(v, o))
c = root.children["LH"]
vc = torch.randn(c.dim, dtype=torch.float64, device="cuda"); oc = torch.empty_like(vc)
out["level2_apply_ms"] = timeit(lambda: c.apply_system_(vc, oc))
leaf = c.children["HH"]
r = torch.randn(leaf.dim, dtype=torch.float64, device="cuda")
out["leaf_solve_ms"] = timeit(lambda: cholesky_solve(leaf.coarse_solve, r))
L3 = h.leaf_factors[1:4]
r3 = torch.randn(3, leaf.dim, 1, dtype=torch.float64, device="cuda")
out["leaf_solve_batch3_ms"] = timeit(lambda: torch.cholesky_solve(r3, L3))
L16 = h.leaf_factors
r16 = torch.randn(16, leaf.dim, 1, dtype=torch.float64, device="cuda")
out["leaf_solve_batch16_ms"] = timeit(lambda: torch.cholesky_solve(r16, L16))
inv = torch.cholesky_inverse(h.leaf_factors[0])
out["leaf_gemv_ms"] = timeit(lambda: inv @ r)
Linv16 = torch.linalg.inv(L16)
out["trimv16_ms"] = timeit(lambda: Linv16.transpose(1,2) @ (Linv16 @ r16))
out["restrict_ms"] = timeit(lambda: restrict(n, v, ("LL","LH","HL","HH")))
out["prolong_ms"] = timeit(lambda: prolong(n, vc, "LH", o, True))
wf = build_projector(g, mode="fast")
y = torch.empty(w.shape[0], dtype=torch.float64, device="cuda")
out["fast_pair_ms"] = timeit(lambda: (wf.forward_(v, y), wf.backward_(y, o)))
out["parity_pair_ms"] = timeit(lambda: (w.forward_(v, y), w.backward_(y, o)))
from paper_1310_0956_b200 import wmg_preconditioner
M = wmg_preconditioner(h)
out["vcycle_ms"] = timeit(lambda: M.apply_(v, o), reps=5)
print(json.dumps(out, indent=1))
