import json, sys, time
import numpy as np, torch
sys.path.insert(0, ".")
from paper_1310_0956_b200 import build_geometry, build_projector, build_wmg_hierarchy, wmg_preconditioner

def timeit(fn, reps=20):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps * 1e3

n, d, m = 256, 363, 180
w = build_projector(build_geometry(n, d, m))
out = {}
for nu in (0, 2):
    h = build_wmg_hierarchy(w, n, 0.0, 3, nu_pre=nu, nu_post=nu)
    v = torch.randn(n * n, dtype=torch.float64, device="cuda"); o = torch.empty_like(v)
    Me = wmg_preconditioner(h, graph=False)
    Mg = wmg_preconditioner(h, graph=True)
    for _ in range(3): Me.apply_(v, o); Mg.apply_(v, o)
    a = Me.apply_(v, o).clone(); b = Mg.apply_(v, o).clone()
    out[f"nu{nu}"] = {"eager_ms": timeit(lambda: Me.apply_(v, o)), "graph_ms": timeit(lambda: Mg.apply_(v, o)),
                      "maxdiff": float((a - b).abs().max())}
print(json.dumps(out, indent=1))
from paper_1310_0956_b200 import SolverConfig, cgls_solve, random_ellipses, add_gaussian_noise
x_ex = random_ellipses(n, 20, seed=1000)
b = add_gaussian_noise(w @ x_ex, 0.01, seed=1500)
wf = build_projector(build_geometry(n, d, m), mode="fast")
res = {}
for nu in (0, 2):
    h = build_wmg_hierarchy(w, n, 0.0, 3, nu_pre=nu, nu_post=nu)
    for graph in (False, True):
        for outer in ("parity", "fast"):
            ww = w if outer == "parity" else wf
            M = wmg_preconditioner(h, graph=graph)
            ts = []
            for rep in range(3):
                torch.cuda.synchronize(); t0 = time.perf_counter()
                xs, rec = cgls_solve(ww, b, precond=M, cfg=SolverConfig(max_iterations=100, residual_tolerance=1e-4))
                torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
            res[f"nu{nu}_graph{int(graph)}_{outer}"] = {"s": ts, "iters": rec.iterations[-1]}
print(json.dumps(res, indent=1))
