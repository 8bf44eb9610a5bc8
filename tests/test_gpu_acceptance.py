"""The reference's acceptance gate (tests/test_acceptance.py, criteria 1, 4, 5,
6, 8) on the GPU path, against the values the reference itself printed for the
160x160 / 400-angle benchmark (pkg/test_output.txt:213-274).  Criteria 2, 3
and 7 are the spectral / property suites (spectral.py, out of scope; the Haar
properties are in test_host_api.py).

SIRT is bit-identical to the reference, so its numbers must match to
rounding.  BiCGStab trajectories are chaotic in the last bit;
the BiCGStab numbers are compared within a tolerance.  The reference fails its
own criteria 5 and 6; here they are checked as "behaves like the reference"."""
import csv
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

NOISE_SEED = 11


def _errs(rec):
    return np.array(rec.rel_err_l2, dtype=np.float64)


def _first_leq(rec, tol):
    hit = np.nonzero(_errs(rec) <= tol)[0]
    return int(rec.iterations[hit[0]]) if hit.size else None


@pytest.fixture(scope="module")
def bench(gpu):
    from paper_1310_0956_b200 import build_geometry, build_projector, shepp_logan
    g = build_geometry(160, 160, 400)
    w = build_projector(g)
    x_ex = shepp_logan(160)
    return g, w, x_ex, w @ x_ex


@pytest.fixture(scope="module")
def noisy_b(bench):
    from paper_1310_0956_b200 import add_noise
    return add_noise(bench[3], 0.01, NOISE_SEED)


@pytest.fixture(scope="module")
def wmg_lam0(bench):
    from paper_1310_0956_b200 import build_wmg_hierarchy, wmg_preconditioner
    return wmg_preconditioner(build_wmg_hierarchy(bench[1], 160, 0.0, 3))


def test_criterion_1_noise_free_benchmark(bench, wmg_lam0):
    """Reference: WMG-BiCGStab <= 2 % at iteration 8, plain BiCGStab at 54,
    SIRT@1000 error 0.0748, and WMG faster in wall clock."""
    from paper_1310_0956_b200 import SolverConfig, bicgstab_solve, normal_operator, sirt_solve
    _, w, x_ex, b = bench
    op = normal_operator(w, 0.0)
    f = w.T @ b
    _, rec_wmg = bicgstab_solve(op, f, precond=wmg_lam0, cfg=SolverConfig(max_iterations=80),
                                x_ex=x_ex)
    k_wmg = _first_leq(rec_wmg, 0.02)
    _, rec_bicg = bicgstab_solve(op, f, cfg=SolverConfig(max_iterations=400), x_ex=x_ex)
    k_bicg = _first_leq(rec_bicg, 0.02)
    _, rec_sirt = sirt_solve(w, b, None, SolverConfig(max_iterations=1000), x_ex=x_ex)
    assert k_wmg == 8
    assert k_bicg is not None and abs(k_bicg - 54) <= 6 and k_bicg >= 3 * k_wmg
    assert abs(rec_sirt.rel_err_l2[-1] - 0.0748) <= 5e-5
    t_wmg = t_bicg = np.inf
    for _ in range(3):
        t0 = time.perf_counter()
        bicgstab_solve(op, f, precond=wmg_lam0, cfg=SolverConfig(max_iterations=k_wmg))
        t_wmg = min(t_wmg, time.perf_counter() - t0)
        t0 = time.perf_counter()
        bicgstab_solve(op, f, cfg=SolverConfig(max_iterations=k_bicg))
        t_bicg = min(t_bicg, time.perf_counter() - t0)
    assert t_wmg < t_bicg, (t_wmg, t_bicg)


@pytest.fixture(scope="module")
def noisy_runs(bench, noisy_b):
    from paper_1310_0956_b200 import (SolverConfig, bicgstab_solve, build_wmg_hierarchy,
                                      normal_operator, sirt_solve, wmg_preconditioner)
    _, w, x_ex, _ = bench
    rec = {}
    _, rec["sirt"] = sirt_solve(w, noisy_b, None,
                                SolverConfig(max_iterations=1000, regularization_lambda=0.001),
                                x_ex=x_ex)
    f10 = w.T @ noisy_b
    op10 = normal_operator(w, 10.0)
    _, rec["bicgstab"] = bicgstab_solve(
        op10, f10, cfg=SolverConfig(max_iterations=100, regularization_lambda=10.0), x_ex=x_ex)
    m10 = wmg_preconditioner(build_wmg_hierarchy(w, 160, 10.0, 3))
    _, rec["wmg"] = bicgstab_solve(
        op10, f10, precond=m10, cfg=SolverConfig(max_iterations=14, regularization_lambda=10.0),
        x_ex=x_ex)
    return rec


def test_criterion_4_noisy_regularized_errors(noisy_runs):
    """Reference: rel-L2 sirt 0.0973, bicgstab 0.0891, wmg 0.0893 (targets
    0.1385 / 0.1074 / 0.1083 +-30 %); rel-Linf 0.1698 > 0.1100 >= 0.1099."""
    l2 = {k: r.rel_err_l2[-1] for k, r in noisy_runs.items()}
    linf = {k: r.rel_err_linf[-1] for k, r in noisy_runs.items()}
    targets = {"sirt": 0.1385, "bicgstab": 0.1074, "wmg": 0.1083}
    assert all(0.7 * targets[k] <= l2[k] <= 1.3 * targets[k] for k in targets), l2
    assert abs(l2["sirt"] - 0.0973) <= 5e-5
    assert abs(l2["bicgstab"] - 0.0891) <= 5e-4 and abs(l2["wmg"] - 0.0893) <= 5e-4
    assert linf["sirt"] > linf["bicgstab"]
    assert abs(linf["sirt"] - 0.1698) <= 5e-5
    assert abs(linf["bicgstab"] - 0.1100) <= 5e-4 and abs(linf["wmg"] - 0.1099) <= 5e-4


def test_criterion_6_regularized_monotonicity_like_reference(noisy_runs):
    """Reference: max rise above the running minimum sirt 0.00 %, bicgstab
    2.28 %, wmg 0.91 % (it fails its own 2 % bound on BiCGStab)."""
    rise = {}
    for k, r in noisy_runs.items():
        e = _errs(r)
        rise[k] = 100.0 * ((e / np.minimum.accumulate(e)).max() - 1.0)
    assert rise["sirt"] <= 0.005
    assert abs(rise["bicgstab"] - 2.28) <= 0.2 and abs(rise["wmg"] - 0.91) <= 0.2


def test_criterion_5_semi_convergence_like_reference(bench, noisy_b, wmg_lam0):
    """Reference: k_opt wmg 5, bicgstab 30, sirt 2254; minima 0.1089 /
    0.0888 / 0.0905 (it fails its own k_opt windows)."""
    from paper_1310_0956_b200 import (SolverConfig, bicgstab_solve, find_kopt, normal_operator,
                                      sirt_solve)
    _, w, x_ex, _ = bench
    op = normal_operator(w, 0.0)
    f = w.T @ noisy_b
    _, rw = bicgstab_solve(op, f, precond=wmg_lam0, cfg=SolverConfig(max_iterations=42),
                           x_ex=x_ex)
    _, rb = bicgstab_solve(op, f, cfg=SolverConfig(max_iterations=300), x_ex=x_ex)
    _, rs = sirt_solve(w, noisy_b, None, SolverConfig(max_iterations=8000), x_ex=x_ex)
    assert find_kopt(rs) == 2254 and abs(_errs(rs).min() - 0.0905) <= 5e-5
    assert find_kopt(rw) == 5 and abs(_errs(rw).min() - 0.1089) <= 5e-4
    assert abs(find_kopt(rb) - 30) <= 2 and abs(_errs(rb).min() - 0.0888) <= 5e-4
    assert find_kopt(rw) < find_kopt(rb) < find_kopt(rs)


def test_criterion_8_bench_determinism(gpu, tmp_path):
    from paper_1310_0956_b200.cli import main
    args = ["bench", "--table", "3", "--n", "32", "--angles", "48", "--detectors", "48",
            "--levels", "3", "--iters-scale", "0.1"]
    outs = [tmp_path / "run1", tmp_path / "run2"]
    for o in outs:
        assert main(args + ["--outdir", str(o)]) == 0

    def numeric(o):
        with open(o / "table3.csv") as fh:
            return [[c for i, c in enumerate(r) if i != 2] for r in csv.reader(fh)]
    assert numeric(outs[0]) == numeric(outs[1])
