"""GPU solvers against the reference (golden) and the oracle restatements.

* sirt_solve: iterates BIT-IDENTICAL to the reference's sirt_solve (config-0
  geometry, 200 iterations; regularised w16 case); logged norms within 1e-12.
* normal_operator: bit-identical to the reference.
* CGLS / BiCGStab / GMRES: bit-identical to oracle/solvers.py (same DET_SUM
  reductions); BiCGStab also within the reference's reordering envelope.
* The reference's own BiCGStab behaviour tests (tests/test_solvers.py:108-167)
  run unchanged against the GPU solver with dense numpy operators.
"""
import numpy as np
import pytest

from conftest import case_geometry

pytestmark = pytest.mark.gpu


def _w(golden, name, **kw):
    from paper_1310_0956_b200.geometry import Geometry, build_projector
    meta, _ = golden
    n, d, angles = case_geometry(meta["projector"][name])
    return build_projector(Geometry(n, d, angles.size, angles=angles), **kw)


def _wo(golden, name):
    from oracle import cproj
    meta, _ = golden
    n, d, angles = case_geometry(meta["projector"][name])
    return cproj.build_csr(n, d, angles)


def test_sirt_cfg0_bitwise_vs_reference(gpu, golden):
    from paper_1310_0956_b200 import SolverConfig, sirt_solve
    _, g = golden
    w = _w(golden, "cfg0")
    x_ex = g["cfg0_phantom"]
    b = w @ x_ex
    x, rec = sirt_solve(w, b, None, SolverConfig(max_iterations=200), x_ex=x_ex)
    assert np.array_equal(x, g["sirt_cfg0_x"])
    np.testing.assert_allclose(rec.rel_residual, g["sirt_cfg0_res"], rtol=1e-12)
    np.testing.assert_allclose(rec.rel_err_l2, g["sirt_cfg0_err"], rtol=1e-12)
    assert rec.iterations == list(range(201)) and rec.status == "max-iterations"


def test_sirt_regularised_bitwise_vs_reference(gpu, golden):
    from paper_1310_0956_b200 import SolverConfig, shepp_logan, sirt_solve
    _, g = golden
    w = _w(golden, "w16")
    x, rec = sirt_solve(w, w @ shepp_logan(16), None,
                        SolverConfig(max_iterations=60, regularization_lambda=0.5))
    assert np.array_equal(x, g["sirt_w16_lam_x"])
    np.testing.assert_allclose(rec.rel_residual, g["sirt_w16_lam_res"], rtol=1e-12)


def test_sirt_conventions(gpu, golden):
    from paper_1310_0956_b200 import SolverConfig, shepp_logan, sirt_solve
    w = _w(golden, "w16")
    ph = shepp_logan(16)
    x, rec = sirt_solve(w, w @ ph, None, SolverConfig(max_iterations=3))
    assert rec.iterations == [0, 1, 2, 3] and rec.rel_residual[0] == 1.0
    assert rec.rel_err_l2[0] is None and rec.status == "max-iterations"
    _, rec = sirt_solve(w, w @ ph, None, SolverConfig(max_iterations=500,
                                                      residual_tolerance=0.5))
    assert rec.status == "converged" and rec.rel_residual[-1] < 0.5
    from paper_1310_0956_b200 import DimensionMismatchError
    with pytest.raises(DimensionMismatchError):
        sirt_solve(w, np.ones(3), None, SolverConfig())


def test_normal_operator_bitwise_vs_reference(gpu, golden):
    from paper_1310_0956_b200 import normal_operator
    _, g = golden
    w = _w(golden, "w16")
    assert np.array_equal(normal_operator(w, 2.5)(g["normal_w16_v"]), g["normal_w16_out"])
    with pytest.raises(ValueError):
        normal_operator(w, -1.0)


@pytest.mark.parametrize("lam,iters", [(0.0, 50), (0.1, 30)])
def test_cgls_cfg0_bitwise_vs_oracle(gpu, golden, lam, iters):
    from oracle import solvers as osol
    from paper_1310_0956_b200 import SolverConfig, cgls_solve
    _, g = golden
    w = _w(golden, "cfg0")
    wo = _wo(golden, "cfg0")
    x_ex = g["cfg0_phantom"]
    b = w @ x_ex
    x, rec = cgls_solve(w, b, cfg=SolverConfig(max_iterations=iters, regularization_lambda=lam),
                        x_ex=x_ex)
    xo, reco = osol.cgls_solve(wo, b, max_iterations=iters, lam=lam, x_ex=x_ex)
    assert np.array_equal(x, xo)
    assert rec.rel_residual == reco.rel_residual
    assert rec.rel_err_l2 == reco.rel_err_l2
    assert rec.rel_residual[-1] < 1e-2


def test_bicgstab_bitwise_vs_oracle_and_reference_envelope(gpu, golden):
    from oracle import solvers as osol
    from paper_1310_0956_b200 import SolverConfig, bicgstab_solve, normal_operator, shepp_logan
    _, g = golden
    w = _w(golden, "w16")
    wo = _wo(golden, "w16")
    ph = shepp_logan(16)
    f = w.T @ (w @ ph)
    x, rec = bicgstab_solve(normal_operator(w, 1.0), f, cfg=SolverConfig(max_iterations=30))
    xo, reco = osol.bicgstab_solve(osol.normal_operator(wo, 1.0), f, max_iterations=30)
    assert np.array_equal(x, xo)
    assert rec.rel_residual == reco.rel_residual
    ref = g["bicg_w16_res"]
    np.testing.assert_allclose(rec.rel_residual[:10], ref[:10], rtol=1e-6)


@pytest.mark.parametrize("precond", [False, True])
def test_gmres_bitwise_vs_oracle(gpu, golden, precond):
    from oracle import solvers as osol
    from paper_1310_0956_b200 import SolverConfig, gmres_solve, normal_operator, shepp_logan
    w = _w(golden, "w16")
    wo = _wo(golden, "w16")
    ph = shepp_logan(16)
    f = w.T @ (w @ ph)
    pre = None
    if precond:
        d = np.asarray(w.T @ (w @ np.ones(256)))
        dinv = 1.0 / d
        pre = lambda v: dinv * np.asarray(v)   # noqa: E731  (host callable, bridged)
    x, rec = gmres_solve(normal_operator(w, 1.0), f, precond=pre,
                         cfg=SolverConfig(max_iterations=25), restart=10, x_ex=ph)
    xo, reco = osol.gmres_solve(osol.normal_operator(wo, 1.0), f, precond=pre,
                                max_iterations=25, restart=10, x_ex=ph)
    assert rec.iterations == reco.iterations
    np.testing.assert_array_equal(rec.rel_residual, reco.rel_residual)
    assert np.array_equal(x, xo)
    assert rec.rel_residual[-1] < 1e-3


# ---- the reference's BiCGStab behaviour tests, run on the GPU solver -------
@pytest.fixture(scope="module")
def spd8():
    rng = np.random.default_rng(7)
    b = rng.standard_normal((8, 8))
    a = b.T @ b + np.eye(8)
    f = rng.standard_normal(8)
    return a, f, np.linalg.solve(a, f)


def test_bicg_matches_direct_solve(gpu, spd8):
    from paper_1310_0956_b200 import SolverConfig, bicgstab_solve
    a, f, x_direct = spd8
    x, rec = bicgstab_solve(lambda v: a @ v, f,
                            cfg=SolverConfig(max_iterations=8, residual_tolerance=1e-10))
    assert rec.status == "converged"
    np.testing.assert_allclose(x, x_direct, atol=1e-10)


def test_bicg_exact_preconditioner(gpu, spd8):
    from paper_1310_0956_b200 import SolverConfig, bicgstab_solve
    a, f, x_direct = spd8
    ainv = np.linalg.inv(a)
    x, rec = bicgstab_solve(lambda v: a @ v, f, precond=lambda v: ainv @ v,
                            cfg=SolverConfig(max_iterations=5, residual_tolerance=1e-12))
    assert rec.status == "converged" and rec.iterations[-1] <= 2
    np.testing.assert_allclose(x, x_direct, atol=1e-9)


def test_bicg_zero_rhs_breakdown_warmstart(gpu, spd8):
    from paper_1310_0956_b200 import DimensionMismatchError, SolverConfig, bicgstab_solve
    a, f, x_direct = spd8
    x, rec = bicgstab_solve(lambda v: a @ v, np.zeros(8))
    assert rec.status == "converged"
    np.testing.assert_array_equal(x, 0.0)
    _, rec = bicgstab_solve(lambda v: np.zeros_like(v), f, cfg=SolverConfig(max_iterations=10))
    assert rec.status == "breakdown"
    x0 = np.arange(1.0, 9.0)
    _, rec = bicgstab_solve(lambda v: a @ v, a @ x0, x0=x0, cfg=SolverConfig(max_iterations=5))
    assert rec.status == "converged" and rec.iterations == [0]
    _, rec = bicgstab_solve(lambda v: a @ v, f, x_ex=x_direct,
                            cfg=SolverConfig(max_iterations=100, residual_tolerance=1e-13))
    assert rec.has_errors and rec.rel_err_l2[-1] < 1e-10
    with pytest.raises(DimensionMismatchError):
        bicgstab_solve(lambda v: a @ v, f, x0=np.ones(3))


def test_bicg_reconstructs_phantom(gpu, golden):
    from paper_1310_0956_b200 import SolverConfig, bicgstab_solve, normal_operator, shepp_logan
    w = _w(golden, "w16")
    ph = shepp_logan(16)
    f = w.T @ (w @ ph)
    _, rec = bicgstab_solve(normal_operator(w, 0.0), f, x_ex=ph,
                            cfg=SolverConfig(max_iterations=400, residual_tolerance=1e-12))
    assert min(rec.rel_err_l2) < 1e-3


def test_device_tensors_stay_on_device(gpu, golden):
    torch = gpu
    from paper_1310_0956_b200 import SolverConfig, cgls_solve
    w = _w(golden, "w16")
    b = torch.from_numpy(np.ones(w.shape[0])).cuda()
    x, rec = cgls_solve(w, b, cfg=SolverConfig(max_iterations=3))
    assert isinstance(x, torch.Tensor) and x.is_cuda


def test_zero_and_degenerate_inputs(gpu, golden):
    """Zero data: every solver returns x = 0 with a converged record at
    iteration 0 (SIRT: zero residual); zero iteration budget is rejected by
    SolverConfig; rays missing the grid (empty rows) do not disturb SIRT."""
    from paper_1310_0956_b200 import (SolverConfig, bicgstab_solve, build_geometry,
                                      build_projector, cgls_solve, gmres_solve,
                                      normal_operator, sirt_solve)
    g = build_geometry(16, 40, 12)          # 40 detectors: many rays miss the 16^2 grid
    w = build_projector(g)
    zb = np.zeros(g.n_data)
    cfg = SolverConfig(max_iterations=5, residual_tolerance=1e-8)
    x, rec = cgls_solve(w, zb, cfg=cfg)
    assert np.all(x == 0) and rec.status == "converged" and rec.iterations == [0]
    x, rec = gmres_solve(normal_operator(w, 0.0), np.zeros(g.n_image), cfg=cfg)
    assert np.all(x == 0) and rec.status == "converged"
    x, rec = bicgstab_solve(normal_operator(w, 0.0), np.zeros(g.n_image), cfg=cfg)
    assert np.all(x == 0) and rec.status == "converged"
    x, rec = sirt_solve(w, zb, None, cfg)
    assert np.all(x == 0)
    with pytest.raises(ValueError):
        SolverConfig(max_iterations=0)
    rs = np.random.default_rng(5)
    xt = rs.uniform(0, 1, g.n_image)
    b = w @ xt
    rows = np.asarray(w.sum(axis=1)).ravel()
    assert (rows == 0).any()                  # empty rows exist
    x, rec = sirt_solve(w, b, None, SolverConfig(max_iterations=50))
    assert np.all(np.isfinite(x)) and rec.rel_residual[-1] < rec.rel_residual[0]


def test_concurrent_cgls_solves_on_two_streams_match_sequential(gpu):
    """Independent slices solved concurrently (host thread + CUDA stream each, a
    projector instance each -- config 4's bench) give bit-identical results."""
    import threading
    torch = gpu
    from paper_1310_0956_b200 import (SolverConfig, build_geometry, build_projector,
                                      cgls_solve, random_ellipses)
    g = build_geometry(256, 363, 180)
    ws = [build_projector(g, precision="float32") for _ in range(2)]
    bs = [torch.from_numpy(ws[0] @ random_ellipses(256, 10, seed=k)).cuda() for k in range(4)]
    cfg = SolverConfig(max_iterations=40, residual_tolerance=1e-6)
    ref = [cgls_solve(ws[0], b, cfg=cfg) for b in bs]
    streams = [torch.cuda.Stream() for _ in range(2)]
    out = [None] * 4

    def worker(i):
        with torch.cuda.stream(streams[i]):
            for k in range(i, 4, 2):
                out[k] = cgls_solve(ws[i], bs[k], cfg=cfg)
        streams[i].synchronize()

    th = [threading.Thread(target=worker, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    torch.cuda.synchronize()
    for k in range(4):
        assert torch.equal(out[k][0], ref[k][0])
        assert out[k][1].rel_residual == ref[k][1].rel_residual


@pytest.mark.parametrize("precond_kind", ["none", "wmg_nu0", "wmg_nu2", "wmg_nograph"])
def test_fused_cgls_kernels_bitwise_vs_unfused(gpu, precond_kind):
    """wmg_cgls_update / wmg_cgls_direction (last reduction level + scalar
    recurrence + vector update in one launch) against the separate
    det_reduce + cgls_scalars + axpy_dev / lincomb_dev kernels: identical
    iterates and records for CGLS and for flexible PCG-NE with the V-cycle
    replayed as its own graph (split) or captured inside the iteration."""
    import torch
    from paper_1310_0956_b200 import (SolverConfig, build_geometry, build_projector,
                                      build_wmg_hierarchy, cgls_solve, random_ellipses,
                                      wmg_preconditioner)
    from paper_1310_0956_b200 import solvers as S
    n, d, m = 64, 91, 90
    w = build_projector(build_geometry(n, d, m), precision="float64", mode="fast")
    b = torch.from_numpy(w @ random_ellipses(n, 10, seed=0)).cuda()
    def run(fused, cfg):
        S.FUSED_CGLS = fused
        try:
            pre = None
            if precond_kind != "none":
                nu = 2 if precond_kind == "wmg_nu2" else 0
                h = build_wmg_hierarchy(w, n, 0.0, 3, nu_pre=nu, nu_post=nu)
                pre = wmg_preconditioner(h, graph=precond_kind != "wmg_nograph")
            x, rec = cgls_solve(w, b, precond=pre, cfg=cfg)
            x2, rec2 = cgls_solve(w, b, precond=pre, cfg=cfg)     # cached graph replay
            assert torch.equal(x, x2) and rec.rel_residual == rec2.rel_residual
            return x, rec
        finally:
            S.FUSED_CGLS = True

    # a fixed iteration count, an early exit on the tolerance, a single iteration
    cfgs = [SolverConfig(max_iterations=20, residual_tolerance=0.0),
            SolverConfig(max_iterations=60, residual_tolerance=1e-3),
            SolverConfig(max_iterations=1, residual_tolerance=0.0)]
    if precond_kind == "none":            # regularised CGLS: delta = <q,q> + lam <p,p>
        cfgs.append(SolverConfig(max_iterations=25, residual_tolerance=0.0,
                                 regularization_lambda=0.1))
    for cfg in cfgs:
        xu, ru = run(False, cfg)
        xf, rf = run(True, cfg)
        assert torch.equal(xf, xu), cfg
        assert rf.rel_residual == ru.rel_residual
        assert rf.status == ru.status and rf.iterations == ru.iterations
        if cfg.residual_tolerance > 0:
            assert ru.status == "converged" and ru.iterations[-1] < cfg.max_iterations


def test_fused_cgls_breakdown_flag(gpu):
    """A non-finite delta = <q,q> (NaN right-hand side): the fused update
    kernel must raise the breakdown flag exactly as wmg_cgls_scalars does, and
    the next solve on the same projector must start clean."""
    import torch
    from paper_1310_0956_b200 import (STATUS_BREAKDOWN, SolverConfig, build_geometry,
                                      build_projector, cgls_solve)
    n, d, m = 32, 47, 20
    w = build_projector(build_geometry(n, d, m), precision="float64", mode="fast")
    b = torch.full((m * d,), float("nan"), dtype=torch.float64, device="cuda")
    _, rec = cgls_solve(w, b, cfg=SolverConfig(max_iterations=5, residual_tolerance=0.0))
    assert rec.status == STATUS_BREAKDOWN
    good = torch.from_numpy(w @ np.ones(n * n)).cuda()
    _, rec = cgls_solve(w, good, cfg=SolverConfig(max_iterations=30, residual_tolerance=1e-6))
    assert rec.rel_residual[-1] < 1e-2 and rec.status != STATUS_BREAKDOWN
