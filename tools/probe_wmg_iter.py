"""Where does a config-1 WMG-CGLS iteration spend its time?  (GPU probe)"""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1310_0956_b200 import (SolverConfig, add_gaussian_noise, build_geometry,  # noqa: E402
                                  build_projector, build_wmg_hierarchy, cgls_solve,
                                  random_ellipses, wmg_preconditioner)


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


def wall(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    return time.perf_counter() - t0, r


n, d, m = 256, 363, 180
g = build_geometry(n, d, m)
w = build_projector(g)
wf = build_projector(g, precision="float64", mode="fast")
x_ex = random_ellipses(n, 20, seed=1000)
b = add_gaussian_noise(w @ x_ex, 0.01, seed=1500)
bd = torch.from_numpy(b).cuda()
out = {}
v = torch.randn(n * n, dtype=torch.float64, device="cuda")
o = torch.empty_like(v)
y = torch.empty(m * d, dtype=torch.float64, device="cuda")
out["fast64_pair_ms"] = ev_time(lambda: (wf.forward_(v, y), wf.backward_(y, o)))
for nu in (0, 2):
    for mode in ("fast", "fast32"):
        t, h = wall(lambda: build_wmg_hierarchy(w, n, 0.0, 3, nu_pre=nu, nu_post=nu,
                                                node_mode=mode))
        M = wmg_preconditioner(h)
        r = {"setup_s": t}
        r["apply1_s"], _ = wall(lambda: M.apply_(v, o))
        r["apply2_s"], _ = wall(lambda: M.apply_(v, o))
        r["apply3_s"], _ = wall(lambda: M.apply_(v, o))
        r["graphed_apply_ms"] = ev_time(lambda: M.apply_(v, o))
        Me = wmg_preconditioner(h, graph=False)
        r["eager_apply_ms"] = ev_time(lambda: Me.apply_(v, o), reps=3)
        cfg = SolverConfig(max_iterations=100, residual_tolerance=1e-4)
        for k in range(2):
            r[f"solve{k}_s"], (_, rec) = wall(lambda: cgls_solve(wf, bd, precond=M, cfg=cfg))
        r["iters"] = rec.iterations[-1]
        out[f"nu{nu}_{mode}"] = r
t, (_, rec) = wall(lambda: cgls_solve(wf, bd, cfg=SolverConfig(max_iterations=500,
                                                                residual_tolerance=1e-4)))
t, (_, rec) = wall(lambda: cgls_solve(wf, bd, cfg=SolverConfig(max_iterations=500,
                                                                residual_tolerance=1e-4)))
out["cgls"] = {"s": t, "iters": rec.iterations[-1]}
print(json.dumps(out, indent=1))
