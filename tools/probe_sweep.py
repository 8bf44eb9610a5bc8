import sys, time, torch
sys.path.insert(0, ".")
from paper_1310_0956_b200 import build_geometry, build_projector
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for n in (256, 512, 768, 1024, 2048, 4096):
    d = int(-(-n * 1.4142135623730951 // 1))
    w = build_projector(build_geometry(n, d, n), precision="float32")
    x = torch.rand(n * n, device="cuda"); y = torch.rand(n * d, device="cuda")
    s, o = torch.empty_like(y), torch.empty_like(x)
    for _ in range(5):
        w.forward_(x, s); w.backward_(y, o)
    res = {}
    for name, fn in (("fwd", lambda: w.forward_(x, s)), ("bwd", lambda: w.backward_(y, o))):
        ts = []
        for _ in range(30 if n < 4096 else 8):
            if n < 4096: flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); fn(); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        ts.sort(); res[name] = ts[len(ts) // 2]
    print(f"n={n} fwd {res['fwd']:.1f} us  bwd {res['bwd']:.1f} us  pair GRays/s {n*d/ (res['fwd']+res['bwd'])/1e3:.3f}", flush=True)
