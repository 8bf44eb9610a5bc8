"""Time wmg_spd_inverse on a batch of SPD matrices (default 16 x 4096^2)."""
import sys
import time
import torch
sys.path.insert(0, ".")
from paper_1310_0956_b200.sparse_kernels import spd_inverse_  # noqa: E402

b = int(sys.argv[1]) if len(sys.argv) > 1 else 16
p = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
r = torch.randn(p, p, dtype=torch.float64, device="cuda") / p ** 0.5
a = (r @ r.T + torch.eye(p, dtype=torch.float64, device="cuda")).expand(b, p, p).contiguous()
x = a.clone()
for i in range(reps):
    x.copy_(a)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    spd_inverse_(x)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"spd_inverse {b}x{p}: {dt*1e3:.2f} ms  {b * p**3 / dt / 1e12:.1f} TF/s (p^3 flops)",
          flush=True)
err = (a[0] @ x[0] - torch.eye(p, dtype=torch.float64, device="cuda")).abs().max().item()
print("max |A X - I| =", err)
