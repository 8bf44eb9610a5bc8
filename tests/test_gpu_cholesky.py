"""Hand-written dense Cholesky factor / solve (csrc/cholesky.cu) against the
reference's cholesky_factor / cholesky_solve (LAPACK potrf / potrs through
scipy; /root/reference/pkg/src/wmgtomo/sparse_kernels.py:53-75), frozen by
``tests/golden/make_chol_golden.py``; plus the reference's own Cholesky unit
tests (tests/test_sparse_kernels.py:41-71) run against the GPU API."""
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
sys.path.insert(0, HERE)


@pytest.fixture(scope="module")
def chol_golden():
    return dict(np.load(os.path.join(HERE, "chol_golden.npz")))


def _kms(p):
    from make_chol_golden import kms
    return kms(p)


@pytest.mark.parametrize("name", ["spd8", "known2", "rand300", "w16leaf"])
def test_factor_and_solve_vs_reference(gpu, chol_golden, name):
    from paper_1310_0956_b200 import cholesky_factor, cholesky_solve
    g = chol_golden
    G, rhs = g[f"{name}_g"], g[f"{name}_rhs"]
    f = cholesky_factor(G)
    L = f.lower
    assert isinstance(L, np.ndarray) and L.shape == G.shape
    assert np.array_equal(np.triu(L, 1), np.zeros_like(L))        # zeros above, as LAPACK
    Lr = g[f"{name}_lower"]
    assert np.linalg.norm(L - Lr) <= 1e-13 * np.linalg.norm(Lr)
    x = cholesky_solve(f, rhs)
    assert isinstance(x, np.ndarray) and x.shape == rhs.shape
    xr = g[f"{name}_x"]
    cond = np.linalg.cond(G)
    assert np.linalg.norm(x - xr) <= 1e-15 * cond * 10 * np.linalg.norm(xr)
    assert np.array_equal(f.solve(rhs), x)                         # deterministic


@pytest.mark.parametrize("p", [512, 1024])
def test_large_factor_and_solve(gpu, chol_golden, p):
    torch = gpu
    from paper_1310_0956_b200 import cholesky_factor, cholesky_solve
    G = _kms(p)
    Gd = torch.from_numpy(G).cuda()
    f = cholesky_factor(Gd)
    L = f.lower
    assert L.is_cuda
    rec = (L @ L.T).cpu().numpy()
    assert np.linalg.norm(rec - G) <= 1e-14 * np.linalg.norm(G)
    rhs = chol_golden[f"kms{p}_rhs"]
    x = cholesky_solve(f, torch.from_numpy(rhs).cuda()).cpu().numpy()
    xr = chol_golden[f"kms{p}_x"]
    assert np.linalg.norm(x - xr) <= 1e-13 * np.linalg.norm(xr)


def test_batched_factor_and_solve(gpu):
    torch = gpu
    from paper_1310_0956_b200 import cholesky_factor, cholesky_solve
    rs = np.random.default_rng(11)
    mats = []
    for _ in range(3):
        a = rs.standard_normal((256, 256))
        mats.append(a @ a.T / 256 + np.eye(256))
    G = torch.from_numpy(np.stack(mats)).cuda()
    f = cholesky_factor(G)
    B = rs.standard_normal((3, 256, 2))
    X = cholesky_solve(f, torch.from_numpy(B).cuda()).cpu().numpy()
    for i in range(3):
        ref = np.linalg.solve(mats[i], B[i])
        assert np.linalg.norm(X[i] - ref) <= 1e-12 * np.linalg.norm(ref)


def test_reference_contract(gpu, chol_golden):
    """tests/test_sparse_kernels.py:41-71 of the reference, on the GPU API."""
    from paper_1310_0956_b200 import (DimensionMismatchError, NotPositiveDefiniteError,
                                      cholesky_factor, cholesky_solve)
    f = cholesky_factor(np.array([[4.0, 2.0], [2.0, 3.0]]))
    assert f.dimension == 2
    np.testing.assert_allclose(f.lower, [[2.0, 0.0], [1.0, np.sqrt(2.0)]], atol=1e-14)
    G, rhs = chol_golden["spd8_g"], chol_golden["spd8_rhs"]
    np.testing.assert_allclose(cholesky_factor(G).solve(rhs), np.linalg.solve(G, rhs),
                               atol=1e-10)
    with pytest.raises(NotPositiveDefiniteError):
        cholesky_factor(np.array([[1.0, 2.0], [0.0, 1.0]]))
    with pytest.raises(NotPositiveDefiniteError):
        cholesky_factor(np.array([[1.0, 0.0], [0.0, -1.0]]))
    with pytest.raises(DimensionMismatchError):
        cholesky_factor(np.ones((2, 3)))
    with pytest.raises(DimensionMismatchError):
        cholesky_factor(G).solve(np.ones(5))
    # the failing leading minor is reported like potrf's info (order 130 > 128:
    # the failure sits in the second pivot block)
    bad = _kms(256)
    bad[129, 129] = -1.0
    with pytest.raises(NotPositiveDefiniteError, match="order 130"):
        cholesky_factor(bad)
    with pytest.raises(ValueError):
        cholesky_solve(f, np.ones((3, 3)))


def test_wmg_leaf_coarse_solve_uses_factor(gpu):
    """DenseFactorization of a WMG leaf: the explicit-inverse GEMV of the
    V-cycle and the Cholesky solve (factor formed on first use) agree."""
    torch = gpu
    from paper_1310_0956_b200 import build_geometry, build_projector, build_wmg_hierarchy
    w = build_projector(build_geometry(16, 24, 24))
    h = build_wmg_hierarchy(w, 16, 1.0, 2)
    leaf = h.root.children["HL"].coarse_solve
    r = torch.from_numpy(np.random.default_rng(5).standard_normal(leaf.dimension)).cuda()
    a = leaf.apply_inverse(r)
    b = leaf.solve(r)
    assert float((a - b).norm()) <= 1e-12 * float(b.norm())
