"""Freeze WMG solver trajectories of the CPU ORACLE (run in the build container):

    python tests/golden/make_wmg_golden.py

The reference has no CGLS / flexible PCG-NE / GMRES and no smoothed V-cycle
(SURVEY.md s8 a16/a17), so these fixtures come from the oracle restatements in
``oracle/`` -- whose smoother-free cycle, BiCGStab and CSR are themselves pinned
to the reference by ``make_golden.py`` / ``tests/test_oracle.py``.  Each case
runs twice:

  * ``det``   the oracle as the GPU runs it: DET_SUM dots and norms;
  * ``blas``  the same run with numpy/BLAS dots (a different summation order):
              the "CPU vs reordered CPU" drift envelope of SURVEY.md s8(c),
              reported beside the GPU-vs-oracle drift.

Cases (seeded synthetic inputs as in bench.py):
  cfg1_nu0   config 1 (256^2, 180 x 363, fp64, 1 % Gaussian noise), WMG-CGLS,
             3 levels, the reference's smoother-free cycle, to 1e-4;
  cfg1_nu22  the same with 2 pre- + 2 post-smoothing sweeps per level;
  cfg2s_gm   downscaled config 2 (256^2, 180 x 363, 50-ellipse phantom
             U[0,1], Poisson I0 = 1e5, mu = 2/n), WMG-GMRES on the normal
             equations, 4 levels, smoother-free, restart 100, to 1e-4.

Writes ``tests/golden/wmg_golden.json`` (histories, omegas, statuses) and
``tests/golden/wmg_golden.npz`` (final iterates).
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.abspath(os.path.join(HERE, "..", ".."))
sys.path.insert(0, ROOT)


def cfg1_data():
    from oracle import cproj
    from paper_1310_0956_b200.phantom import add_gaussian_noise, random_ellipses
    n, d, m = 256, 363, 180
    w = cproj.build_csr(n, d, cproj.equiangular(m))
    x_ex = random_ellipses(n, 20, seed=1000)
    b = add_gaussian_noise(cproj.csr_matvec(w, x_ex), 0.01, seed=1500)
    return n, w, x_ex, b


def cfg2s_data():
    from oracle import cproj
    from paper_1310_0956_b200.phantom import poisson_log_data, random_ellipses
    n, d, m = 256, 363, 180
    w = cproj.build_csr(n, d, cproj.equiangular(m))
    x_ex = random_ellipses(n, 50, seed=2000, value_range=(0.0, 1.0))
    b = poisson_log_data(cproj.csr_matvec(w, x_ex), 1e5, 2.0 / n, seed=2500)
    return n, w, x_ex, b


class _BlasDots:
    """Swap the oracle's DET_SUM reductions for BLAS-ordered ones."""

    def __enter__(self):
        from oracle import solvers as osol
        self.saved = {k: getattr(osol, k) for k in ("det_sum", "det_dot", "det_sq",
                                                    "det_norm")}
        osol.det_sum = lambda v: float(np.sum(np.asarray(v, dtype=np.float64)))
        osol.det_dot = lambda a, b: float(np.dot(a, b))
        osol.det_sq = lambda a: float(np.dot(a, a))
        osol.det_norm = lambda a: float(np.sqrt(np.dot(a, a)))
        return self

    def __exit__(self, *exc):
        from oracle import solvers as osol
        for k, v in self.saved.items():
            setattr(osol, k, v)


def _omegas(root):
    from oracle import multilevel as oml
    return {nd.path or "root": nd.omega for nd in oml._nodes(root) if nd.lower is None}


def run_cgls(n, w, x_ex, b, nu):
    from oracle import multilevel as oml
    from oracle import solvers as osol
    t0 = time.perf_counter()
    root = oml.build_hierarchy(w, n, 0.0, 3, nu_pre=nu, nu_post=nu)
    t1 = time.perf_counter()
    x, rec = osol.cgls_solve(w, b, precond=oml.preconditioner(root), max_iterations=100,
                             tol=1e-4, x_ex=x_ex)
    t2 = time.perf_counter()
    return root, x, rec, (t1 - t0, t2 - t1)


def run_gmres(n, w, x_ex, b, levels):
    from oracle import multilevel as oml
    from oracle import solvers as osol
    t0 = time.perf_counter()
    root = oml.build_hierarchy(w, n, 0.0, levels)
    t1 = time.perf_counter()
    op = osol.normal_operator(w, 0.0)
    f = w.T @ b
    x, rec = osol.gmres_solve(op, f, precond=oml.preconditioner(root), max_iterations=300,
                              tol=1e-4, x_ex=x_ex, restart=100)
    t2 = time.perf_counter()
    return root, x, rec, (t1 - t0, t2 - t1)


def _rec(rec):
    return {"iterations": rec.iterations, "rel_residual": rec.rel_residual,
            "rel_err_l2": rec.rel_err_l2, "status": rec.status}


def _drift(a, b):
    a, b = np.asarray(a), np.asarray(b)
    k = min(a.size, b.size)
    return [float(abs(a[i] - b[i]) / abs(a[i])) for i in range(k)]


def main():
    from oracle import cproj
    cproj.set_threads(os.cpu_count() or 1)
    meta, arrays = {}, {}
    n, w, x_ex, b = cfg1_data()
    arrays["cfg1_b"] = b
    for nu, name in ((0, "cfg1_nu0"), (2, "cfg1_nu22")):
        root, x, rec, secs = run_cgls(n, w, x_ex, b, nu)
        with _BlasDots():
            root_b, x_b, rec_b, _ = run_cgls(n, w, x_ex, b, nu)
        meta[name] = {"det": _rec(rec), "blas": _rec(rec_b), "omega": _omegas(root),
                      "omega_blas": _omegas(root_b),
                      "envelope_rel_residual": _drift(rec.rel_residual, rec_b.rel_residual),
                      "envelope_x": float(np.linalg.norm(x - x_b) / np.linalg.norm(x)),
                      "oracle_seconds": {"setup": secs[0], "solve": secs[1]},
                      "levels": 3, "nu_pre": nu, "nu_post": nu, "lambda": 0.0}
        arrays[f"{name}_x"] = x
        print(name, rec.iterations[-1], rec.status, rec.rel_residual[-1], secs,
              max(meta[name]["envelope_rel_residual"]), flush=True)
    n, w, x_ex, b = cfg2s_data()
    arrays["cfg2s_b"] = b
    root, x, rec, secs = run_gmres(n, w, x_ex, b, 4)
    with _BlasDots():
        _, x_b, rec_b, _ = run_gmres(n, w, x_ex, b, 4)
    meta["cfg2s_gm"] = {"det": _rec(rec), "blas": _rec(rec_b),
                        "envelope_rel_residual": _drift(rec.rel_residual, rec_b.rel_residual),
                        "envelope_x": float(np.linalg.norm(x - x_b) / np.linalg.norm(x)),
                        "oracle_seconds": {"setup": secs[0], "solve": secs[1]},
                        "levels": 4, "restart": 100, "lambda": 0.0}
    arrays["cfg2s_gm_x"] = x
    print("cfg2s_gm", rec.iterations[-1], rec.status, rec.rel_residual[-1], secs,
          max(meta["cfg2s_gm"]["envelope_rel_residual"]), flush=True)
    with open(os.path.join(HERE, "wmg_golden.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    np.savez_compressed(os.path.join(HERE, "wmg_golden.npz"), **arrays)


if __name__ == "__main__":
    main()
