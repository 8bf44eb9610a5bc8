"""Batched GEMV bandwidth (16 leaf inverses of 4096^2, the config-1 V-cycle's coarse solves)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1310_0956_b200.sparse_kernels import batched_gemv  # noqa: E402

A = torch.rand(16, 4096, 4096, dtype=torch.float64, device="cuda")
x = torch.rand(16, 4096, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
for b in (1, 3, 16):
    batched_gemv(A[:b], x[:b], out=y[:b])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        batched_gemv(A[:b], x[:b], out=y[:b])
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 20 / 1e3
    print(f"batch {b}: {t * 1e6:.1f} us, {b * 4096 * 4096 * 8 / t / 1e12:.2f} TB/s")
ref = torch.bmm(A, x.unsqueeze(-1)).squeeze(-1)
batched_gemv(A, x, out=y)
print("max rel err", float(((y - ref).abs().max() / ref.abs().max())))
