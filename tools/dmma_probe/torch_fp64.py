"""cuBLAS DGEMM / cuSOLVER rates at the leaf size (4096) on B200."""
import time, torch
def t(fn, r=3):
    fn(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(r): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / r
n = 4096
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
s = t(lambda: a @ b); print(f"dgemm {n}: {2*n**3/s/1e12:.1f} TF ({s*1e3:.1f} ms)")
g = a @ a.T + n * torch.eye(n, dtype=torch.float64, device="cuda")
G = g.unsqueeze(0).repeat(16, 1, 1)
s = t(lambda: torch.linalg.cholesky_ex(G)); print(f"chol 16x{n}: {s*1e3:.1f} ms")
L = torch.linalg.cholesky(G)
s = t(lambda: torch.cholesky_inverse(L)); print(f"cholesky_inverse 16x{n}: {s*1e3:.1f} ms")
I = torch.eye(n, dtype=torch.float64, device="cuda").expand(16, n, n)
s = t(lambda: torch.linalg.solve_triangular(L, I, upper=False)); print(f"trsm(L,I) 16x{n}: {s*1e3:.1f} ms")
s = t(lambda: torch.linalg.inv_ex(G)); print(f"inv_ex 16x{n}: {s*1e3:.1f} ms")
