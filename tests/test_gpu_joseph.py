"""Joseph interpolating kernel on the B200: the parity
kernels built on JosephWalker / jbwd_kernel reproduce the reference's
build_projector(kernel="joseph") (geometry.py:131-175) bit for bit -- CSR,
W x (csr_matvec order), W^T y (csc_matvec order), row and column sums -- and
the solvers / WMG hierarchy accept a Joseph projector."""
import hashlib

import numpy as np
import pytest

from conftest import case_geometry, case_vectors

pytestmark = pytest.mark.gpu

CASES = ["jos_tiny_vertical", "jos_tiny_two", "jos_diag8", "jos_miss12", "jos_odd15",
         "jos_w16", "jos_cfg0", "jos_cfg1", "jos_bench160"]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _proj(spec):
    from paper_1310_0956_b200.geometry import Geometry, build_projector
    n, d, angles = case_geometry(spec)
    return build_projector(Geometry(n, d, angles.size, angles=angles), kernel="joseph")


@pytest.mark.parametrize("name", CASES)
def test_joseph_bitwise_vs_reference(gpu, golden, name):
    torch = gpu
    meta, _ = golden
    spec = meta["joseph"][name]
    w = _proj(spec)
    assert w.kernel == "joseph"
    indptr, cols, vals, _ = w.csr_device()
    assert int(indptr[-1]) == spec["nnz"]
    assert sha(indptr.cpu().numpy()) == spec["indptr"]
    assert sha(cols.cpu().numpy()) == spec["indices"]
    assert sha(vals.cpu().numpy()) == spec["data"]
    x, y = case_vectors(spec, w.shape[0])
    wx = torch.empty(w.shape[0], dtype=torch.float64, device="cuda")
    wty = torch.empty(w.shape[1], dtype=torch.float64, device="cuda")
    w.forward_(torch.from_numpy(x).cuda(), wx)
    w.backward_(torch.from_numpy(y).cuda(), wty)
    assert sha(wx.cpu().numpy()) == spec["wx"]
    assert sha(wty.cpu().numpy()) == spec["wty"]
    assert sha(w.row_sums_dev().cpu().numpy()) == spec["rows"]
    assert sha(w.col_sums_dev().cpu().numpy()) == spec["cols"]


def test_joseph_modes_and_errors(gpu):
    from paper_1310_0956_b200 import build_geometry, build_projector
    g = build_geometry(16, 24, 24)
    with pytest.raises(ValueError):
        build_projector(g, kernel="joseph", precision="float32")
    with pytest.raises(ValueError):
        build_projector(g, kernel="joseph", mode="fast")
    with pytest.raises(ValueError):
        build_projector(g, kernel="bogus")


def test_joseph_solvers_and_wmg(gpu, golden, oracle_proj):
    """SIRT on a Joseph W is bit-identical to the oracle restatement; WMG-CGLS
    (exact leaf factors + parity node systems) converges."""
    from oracle import solvers as osol
    from paper_1310_0956_b200 import (SolverConfig, build_wmg_hierarchy, cgls_solve,
                                      shepp_logan, sirt_solve, wmg_preconditioner)
    meta, _ = golden
    spec = meta["joseph"]["jos_w16"]
    n, d, angles = case_geometry(spec)
    w = _proj(spec)
    ph = shepp_logan(16)
    b = w @ ph
    wc = oracle_proj.build_csr(n, d, angles, kernel="joseph")
    assert np.array_equal(b, oracle_proj.csr_matvec(wc, ph))
    x, rec = sirt_solve(w, b, None, SolverConfig(max_iterations=40), x_ex=ph)
    xo, reco = osol.sirt_solve(wc, b, None, 40, x_ex=ph)
    assert np.array_equal(x, xo)
    cfg = SolverConfig(max_iterations=60, residual_tolerance=1e-8, regularization_lambda=0.1)
    h = build_wmg_hierarchy(w, 16, 0.1, 2)
    _, r = cgls_solve(w, b, precond=wmg_preconditioner(h), cfg=cfg)
    _, r0 = cgls_solve(w, b, cfg=cfg)
    assert r.status == "converged" and r.iterations[-1] < r0.iterations[-1]
