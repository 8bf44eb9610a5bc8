"""Where does WMG setup time go?  Config 1 (256^2, 3 levels) and config 2
(1024^2, 5 levels): leaf Grams, batched Cholesky, inverse, smoothers, capture."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1310_0956_b200 import build_geometry, build_projector, wmg_preconditioner  # noqa
from paper_1310_0956_b200 import multilevel as ML  # noqa: E402


def tic():
    torch.cuda.synchronize()
    return time.perf_counter()


def run(n, d, m, levels, nu, prec):
    dev = torch.device("cuda", 0)
    w = build_projector(build_geometry(n, d, m), precision=prec, device=dev)
    for rep in range(2):
        t0 = tic()
        paths, grams = ML._assemble_leaf_grams(w, n, 0.0, levels)
        t1 = tic()
        g16 = grams[:min(16, len(grams))]
        low, info = torch.linalg.cholesky_ex(g16)
        t2 = tic()
        from paper_1310_0956_b200.sparse_kernels import spd_inverse_
        spd_inverse_(g16)
        t3 = tic()
        del low, grams
        torch.cuda.empty_cache()
        t4 = tic()
        h = ML.build_wmg_hierarchy(w, n, 0.0, levels, nu_pre=nu, nu_post=nu)
        t5 = tic()
        M = wmg_preconditioner(h)
        M.prepare() if hasattr(M, "prepare") else None
        t6 = tic()
        print(f"n={n} L={levels} rep={rep}: grams {t1-t0:.4f}  chol(<=16) {t2-t1:.4f}  "
              f"sweep-inverse(<=16) {t3-t2:.4f}  full-hierarchy {t5-t4:.4f}  precond+capture {t6-t5:.4f}",
              flush=True)
        del h, M
        torch.cuda.empty_cache()


run(256, 363, 180, 3, 2, "float64")
if len(sys.argv) > 1:
    run(1024, 1449, 720, 5, 0, "float32")
