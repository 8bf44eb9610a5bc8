"""Dense GEMV vs packed symmetric GEMV on 16 x 4096^2 leaf inverses (one and
three matrices per call, as the V-cycle issues them)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_1310_0956_b200.sparse_kernels import PackedSymmetric, batched_gemv  # noqa: E402

p = 4096
r = torch.randn(p, p, dtype=torch.float64, device="cuda")
a = (r + r.T).expand(16, p, p).contiguous()
pk = PackedSymmetric.pack(a)
x = torch.randn(16, p, dtype=torch.float64, device="cuda")


def ev(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for nb in (1, 3, 16):
    td = ev(lambda: batched_gemv(a[:nb], x[:nb]))
    tp = ev(lambda: batched_gemv(pk[:nb], x[:nb]))
    bd, bp = nb * p * p * 8, nb * pk.data.shape[1] * 8
    print(f"batch {nb:2d}: dense {td:7.1f} us ({bd / td / 1e3:6.0f} GB/s)   packed {tp:7.1f} us "
          f"({bp / tp / 1e3:6.0f} GB/s)")
y1, y2 = batched_gemv(a, x), batched_gemv(pk, x)
print("max rel diff", ((y1 - y2).abs().max() / y1.abs().max()).item())
