"""The REFERENCE's own solver code driven by the GPU operators (the drop-in claim
of INTEGRATION.md).

``wmgtomo`` is the unmodified reference package, installed offline into the
git-ignored ``baseline/_ref`` (``pip install --no-index --target baseline/_ref``;
it travels to the GPU box with the repo snapshot; the test skips without it).
Its ``sirt_solve`` / ``normal_operator`` / ``bicgstab_solve``
(/root/reference/pkg/src/wmgtomo/solvers.py:95-243) and ``apply`` /
``apply_transpose`` (geometry.py:200-215) run unchanged on a ``LineProjector``
(``shape``, ``@``, ``.T``, ``.tocsr()``, ``.sum(axis)``) and with the GPU
``wmg_preconditioner`` as their ``precond`` callable, and their results are
compared with the golden results the reference produced on its own scipy CSR
(``tests/golden/make_golden.py``).
"""
import os
import sys

import numpy as np
import pytest

from conftest import case_geometry

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def wmgtomo():
    if not os.path.isdir(os.path.join(REF, "wmgtomo")):
        pytest.skip("reference not installed in baseline/_ref")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import wmgtomo as ref
    import wmgtomo.geometry  # noqa: F401
    import wmgtomo.solvers  # noqa: F401
    return ref


def _w(golden, name):
    from paper_1310_0956_b200.geometry import Geometry, build_projector
    meta, _ = golden
    n, d, angles = case_geometry(meta["projector"][name])
    return build_projector(Geometry(n, d, angles.size, angles=angles))


def test_reference_sirt_on_gpu_operator_bitwise(gpu, golden, wmgtomo):
    """Reference sirt_solve + GPU W: the iterate is bit-identical to the
    reference's own run on its CSR (config-0 geometry, 200 iterations)."""
    S = wmgtomo.solvers
    _, g = golden
    w = _w(golden, "cfg0")
    x_ex = g["cfg0_phantom"]
    b = wmgtomo.geometry.apply(w, x_ex)
    x, rec = S.sirt_solve(w, b, None, S.SolverConfig(max_iterations=200), x_ex=x_ex)
    assert np.array_equal(x, g["sirt_cfg0_x"])
    assert np.array_equal(np.asarray(rec.rel_residual), g["sirt_cfg0_res"])
    assert rec.status == "max-iterations"


def test_reference_bicgstab_normal_operator_on_gpu(gpu, golden, wmgtomo):
    """Reference bicgstab_solve(normal_operator(W_gpu)) on w16: bit-identical
    history and iterate to the reference's run on its CSR."""
    S = wmgtomo.solvers
    _, g = golden
    w = _w(golden, "w16")
    from paper_1310_0956_b200 import shepp_logan
    ph = shepp_logan(16)
    f = wmgtomo.geometry.apply_transpose(w, wmgtomo.geometry.apply(w, ph))
    op = S.normal_operator(w, 1.0)
    assert np.array_equal(S.normal_operator(w, 2.5)(g["normal_w16_v"]), g["normal_w16_out"])
    x, rec = S.bicgstab_solve(op, f, cfg=S.SolverConfig(max_iterations=30))
    assert np.array_equal(np.asarray(rec.rel_residual), g["bicg_w16_res"])
    assert np.array_equal(x, g["bicg_w16_x"])


@pytest.mark.parametrize("levels", [2, 3])
def test_reference_bicgstab_with_gpu_wmg_preconditioner(gpu, golden, wmgtomo, levels):
    """Reference bicgstab_solve with the GPU WMG V-cycle as ``precond`` (matrix-
    free node systems, DMMA leaf inverses): within 1e-9 of the reference's
    WMG-BiCGStab history on its own hierarchy."""
    S = wmgtomo.solvers
    _, g = golden
    meta, _ = golden
    from paper_1310_0956_b200 import build_wmg_hierarchy, shepp_logan, wmg_preconditioner
    w = _w(golden, "w16")
    ph = shepp_logan(16)
    f = w.T @ (w @ ph)
    M = wmg_preconditioner(build_wmg_hierarchy(w, 16, 1.0, levels))
    x, rec = S.bicgstab_solve(S.normal_operator(w, 1.0), f, precond=M,
                              cfg=S.SolverConfig(max_iterations=20, residual_tolerance=1e-10))
    ref = g[f"wmgbicg_w16_l{levels}_res"]
    assert rec.status == meta["solvers"][f"wmgbicg_w16_l{levels}_status"]
    assert len(rec.rel_residual) == ref.size
    # early entries: relative agreement; entries near the 1e-10 floor: absolute
    np.testing.assert_allclose(rec.rel_residual, ref, rtol=1e-6, atol=1e-14)
    xr = g[f"wmgbicg_w16_l{levels}_x"]
    assert np.linalg.norm(x - xr) <= 1e-9 * np.linalg.norm(xr)
