"""Freeze the REFERENCE's dense Cholesky factor / solve (run in the build
container, where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_chol_golden.py

Writes ``tests/golden/chol_golden.npz``: for each case the matrix G, the
right-hand side(s), wmgtomo.sparse_kernels.cholesky_factor(G).lower
(scipy/LAPACK potrf) and cholesky_solve(f, rhs) (cho_solve = potrs)
(/root/reference/pkg/src/wmgtomo/sparse_kernels.py:53-75).  Cases: the
reference's own spd8 fixture (tests/conftest.py:23-29), the 2 x 2 known factor
of tests/test_sparse_kernels.py:41-46, a random SPD matrix of order 300
(padded to 384 on the GPU), exactly representable SPD matrices of orders 512
(three right-hand sides) and 1024 (``kms``; rebuilt by the test, only the
solutions stored),
and the w16 two-level WMG leaf Gram of the LL band.
"""
from __future__ import annotations

import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def kms(p):
    """Kac-Murdock-Szego matrix 0.5^|i-j| plus diag((i mod 7) / 8): SPD and
    exactly representable (powers of two), so every host builds it bitwise."""
    i = np.arange(p)
    g = np.ldexp(1.0, -np.abs(i[:, None] - i[None, :]))
    return g + np.diag((i % 7) / 8.0)


def main():
    from wmgtomo.geometry import build_geometry, build_projector
    from wmgtomo.multilevel import build_intergrid_set
    from wmgtomo.sparse_kernels import cholesky_factor, cholesky_solve, spgemm
    arrays = {}

    def case(name, g, rhs):
        f = cholesky_factor(g)
        arrays[f"{name}_g"] = g
        arrays[f"{name}_rhs"] = rhs
        arrays[f"{name}_lower"] = f.lower
        arrays[f"{name}_x"] = cholesky_solve(f, rhs)

    rng = np.random.default_rng(7)                 # the reference's spd8 fixture
    b = rng.standard_normal((8, 8))
    case("spd8", b.T @ b + np.eye(8), rng.standard_normal(8))
    case("known2", np.array([[4.0, 2.0], [2.0, 3.0]]), np.array([1.0, -1.0]))
    rs = np.random.default_rng(300)
    a = rs.standard_normal((300, 300))
    case("rand300", a @ a.T / 300 + 0.1 * np.eye(300), rs.standard_normal(300))
    for p, k in ((512, 3), (1024, 1)):
        rs = np.random.default_rng(p)
        rhs = rs.standard_normal(p) if k == 1 else rs.standard_normal((p, k))
        case(f"kms{p}", kms(p), rhs)
        # large cases: G is regenerated exactly by the test, only x is stored
        del arrays[f"kms{p}_g"], arrays[f"kms{p}_lower"]
    w = build_projector(build_geometry(16, 24, 24))
    s = build_intergrid_set(16)
    pl = spgemm(w, s["LL"].T)
    g = (pl.T @ pl).toarray() + np.eye(64)
    case("w16leaf", g, np.random.default_rng(3).standard_normal((64, 2)))
    np.savez_compressed(os.path.join(HERE, "chol_golden.npz"), **arrays)
    print("wrote", os.path.join(HERE, "chol_golden.npz"))


if __name__ == "__main__":
    main()
