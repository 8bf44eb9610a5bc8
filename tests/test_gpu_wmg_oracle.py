"""WMG-preconditioned Krylov solves on the B200 against the CPU oracle at the
BASELINE configurations they are measured on.

Fixtures: ``tests/golden/make_wmg_golden.py`` runs the oracle restatements
(``oracle/multilevel.py``: reference hierarchy of stored sparse factors, exact
dense Cholesky leaves, the wavelet V-cycle of multilevel.py:175-198 plus the
deterministic SIRT-type smoother; ``oracle/solvers.py``: flexible PCG-NE and
GMRES with DET_SUM reductions) and a BLAS-dot rerun of the same oracle, whose
difference is the CPU-vs-reordered-CPU drift envelope.

The GPU runs its own pipeline: exact W (parity kernels) outside, matrix-free
node systems (fast float64 pair, <= 1e-12), sparse leaf Grams, DMMA SPD
inverses, graphed cycle.  Asserted: identical iteration counts and statuses,
residual histories and errors within 1e-8 relative at every iteration, final
reconstructions within 1e-8, smoother weights omega_p within 1e-10; the
measured GPU drift is printed next to the oracle's own reorder envelope.
"""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def wmg_golden():
    with open(os.path.join(HERE, "wmg_golden.json")) as fh:
        meta = json.load(fh)
    return meta, dict(np.load(os.path.join(HERE, "wmg_golden.npz")))


def _rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return np.abs(a - b) / np.abs(b)


def _check(rec, x, ref, x_ref, tol=1e-8):
    det = ref["det"]
    assert rec.status == det["status"]
    assert rec.iterations == det["iterations"]
    drift = _rel(rec.rel_residual, det["rel_residual"])
    env = np.asarray(ref["envelope_rel_residual"])
    print(f"\n  iterations {rec.iterations[-1]}  max GPU-vs-oracle drift {drift.max():.2e}"
          f"  oracle reorder envelope {env.max():.2e}")
    assert drift.max() <= tol, drift
    assert _rel(rec.rel_err_l2, det["rel_err_l2"]).max() <= tol
    assert np.linalg.norm(x - x_ref) <= tol * np.linalg.norm(x_ref)


@pytest.mark.parametrize("outer", ["parity", "fast"])
@pytest.mark.parametrize("nu", [0, 2])
def test_wmg_cgls_config1_vs_oracle(gpu, wmg_golden, nu, outer):
    """``outer="fast"`` is the bench's pipeline (fast float64 outer pair)."""
    from paper_1310_0956_b200 import (SolverConfig, build_geometry, build_projector,
                                      build_wmg_hierarchy, cgls_solve, random_ellipses,
                                      wmg_preconditioner)
    meta, arr = wmg_golden
    ref = meta["cfg1_nu0" if nu == 0 else "cfg1_nu22"]
    n = 256
    w = build_projector(build_geometry(n, 363, 180))
    x_ex = random_ellipses(n, 20, seed=1000)
    b = arr["cfg1_b"]
    h = build_wmg_hierarchy(w, n, 0.0, 3, nu_pre=nu, nu_post=nu)
    if nu:
        for nd in h.nodes():
            if not nd.is_coarsest:
                om = ref["omega"][nd.path or "root"]
                assert abs(nd.smooth_omega - om) <= 1e-10 * om, nd.path
    wo = w if outer == "parity" else build_projector(build_geometry(n, 363, 180),
                                                     precision="float64", mode="fast")
    x, rec = cgls_solve(wo, b, precond=wmg_preconditioner(h), x_ex=x_ex,
                        cfg=SolverConfig(max_iterations=100, residual_tolerance=1e-4))
    _check(rec, x, ref, arr["cfg1_nu0_x" if nu == 0 else "cfg1_nu22_x"])


def test_wmg_gmres_downscaled_config2_vs_oracle(gpu, wmg_golden):
    from paper_1310_0956_b200 import (SolverConfig, build_geometry, build_projector,
                                      build_wmg_hierarchy, gmres_solve, normal_operator,
                                      random_ellipses, wmg_preconditioner)
    meta, arr = wmg_golden
    ref = meta["cfg2s_gm"]
    n = 256
    w = build_projector(build_geometry(n, 363, 180))
    x_ex = random_ellipses(n, 50, seed=2000, value_range=(0.0, 1.0))
    b = arr["cfg2s_b"]
    M = wmg_preconditioner(build_wmg_hierarchy(w, n, 0.0, 4))
    x, rec = gmres_solve(normal_operator(w, 0.0), w.T @ b, precond=M, x_ex=x_ex, restart=100,
                         cfg=SolverConfig(max_iterations=300, residual_tolerance=1e-4))
    _check(rec, x, ref, arr["cfg2s_gm_x"])


def test_wmg_gmres_downscaled_config2_fp32_pipeline(gpu, wmg_golden):
    """The config-2 pipeline as bench.py runs it (float32 projector, float64
    Krylov vectors, fp32 node systems) against the float64 oracle: same
    iteration count, history within the fp32 projector's error propagation."""
    from paper_1310_0956_b200 import (SolverConfig, build_geometry, build_projector,
                                      build_wmg_hierarchy, gmres_solve, normal_operator,
                                      random_ellipses, wmg_preconditioner)
    meta, arr = wmg_golden
    ref = meta["cfg2s_gm"]
    n = 256
    g = build_geometry(n, 363, 180)
    w32 = build_projector(g, precision="float32")
    x_ex = random_ellipses(n, 50, seed=2000, value_range=(0.0, 1.0))
    b = arr["cfg2s_b"]
    M = wmg_preconditioner(build_wmg_hierarchy(build_projector(g), n, 0.0, 4,
                                               node_mode="fast32"))
    x, rec = gmres_solve(normal_operator(w32, 0.0), w32.T @ b, precond=M, x_ex=x_ex,
                         restart=100,
                         cfg=SolverConfig(max_iterations=300, residual_tolerance=1e-4))
    det = ref["det"]
    assert rec.status == det["status"]
    assert abs(rec.iterations[-1] - det["iterations"][-1]) <= 1
    k = min(len(rec.rel_residual), len(det["rel_residual"]))
    drift = _rel(rec.rel_residual[:k], det["rel_residual"][:k])
    print(f"\n  fp32 pipeline: iterations {rec.iterations[-1]} vs {det['iterations'][-1]},"
          f" max drift {drift.max():.2e}")
    assert drift.max() <= 1e-3
    assert abs(rec.rel_err_l2[-1] - det["rel_err_l2"][-1]) <= 1e-4
