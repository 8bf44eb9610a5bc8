"""Does the n=4096 pair bench slow the following config-1 WMG-CGLS timing?"""
import sys
import time
import torch
sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1310_0956_b200 import build_geometry, build_projector  # noqa: E402

dev = torch.device("cuda", 0)
def show(tag, r):
    print(tag, {kk: round(r[kk], 4) for kk in ("seconds", "setup_seconds", "cgls_seconds")},
          round(r["nu0"]["seconds"], 4), flush=True)

show("fresh", bench.run_wmg_cgls(dev))
n, d, m = bench.workload(4096)
w = build_projector(build_geometry(n, d, m), precision="float32", device=dev)
x = torch.rand(n * n, device=dev)
y = torch.rand(m * d, device=dev)
s = torch.empty(m * d, device=dev)
o = torch.empty(n * n, device=dev)
for _ in range(20):
    w.forward_(x, s)
    w.backward_(y, o)
torch.cuda.synchronize()
show("after_pair", bench.run_wmg_cgls(dev))
time.sleep(5)
show("after_sleep", bench.run_wmg_cgls(dev))
del w, x, y, s, o
torch.cuda.empty_cache()
show("after_free", bench.run_wmg_cgls(dev))
