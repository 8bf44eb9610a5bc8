"""The CPU oracle is pinned to the reference before it is trusted.

Every projector case frozen by tests/golden/make_golden.py (reference CSR
hashes, W x / W^T y / row / column sums on seeded vectors) must be reproduced
bit for bit by oracle/wmg_oracle.c, and the oracle's SIRT restatement must
reproduce the reference trajectory.
"""
import hashlib

import numpy as np
import pytest

from conftest import case_geometry, case_vectors


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


SMALL = ["tiny_vertical", "tiny_two", "diag8", "miss12", "w16", "w40", "cfg0", "cfg1",
         "bench160", "cfg3_512_sub", "cfg3_1024_sub"]
LARGE = ["cfg3_2048_sub", "cfg3_4096_sub"]


@pytest.mark.parametrize("name", SMALL + LARGE)
def test_oracle_csr_matches_reference(golden, oracle_proj, name):
    meta, _ = golden
    spec = meta["projector"][name]
    n, d, angles = case_geometry(spec)
    w, dups = oracle_proj.build_csr(n, d, angles, return_dups=True)
    assert dups == 0
    assert w.nnz == spec["nnz"]
    assert sha(w.indptr.astype(np.int64)) == spec["indptr"]
    assert sha(w.indices.astype(np.int64)) == spec["indices"]
    assert sha(w.data) == spec["data"]
    x, y = case_vectors(spec, w.shape[0])
    assert sha(oracle_proj.csr_matvec(w, x)) == spec["wx"]
    if name not in LARGE:
        assert sha(oracle_proj.forward(n, d, angles, x)) == spec["wx"]
        assert sha(oracle_proj.backward(n, d, angles, y)) == spec["wty"]
    assert sha(w.T @ y) == spec["wty"]
    assert sha(oracle_proj.row_sums(w)) == spec["rows"]
    assert sha(oracle_proj.col_sums(w)) == spec["cols"]


def test_oracle_edge_semantics(oracle_proj):
    # axis-aligned rays: unit weights; central ray on a grid line goes right/up
    w = oracle_proj.build_csr(4, 5, np.array([0.0, np.pi / 2])).toarray()
    assert set(np.unique(w)) <= {0.0, 1.0}
    central_vertical = w[2].reshape(4, 4)
    assert central_vertical[:, 2].sum() == 4.0 and central_vertical[:, 1].sum() == 0.0
    central_horizontal = w[5 + 2].reshape(4, 4)
    assert central_horizontal[1].sum() == 4.0 and central_horizontal[2].sum() == 0.0
    # rays missing the grid are empty rows
    w = oracle_proj.build_csr(4, 12, np.array([0.0]))
    counts = np.diff(w.indptr)
    assert counts[0] == 0 and counts[-1] == 0 and counts[4:8].min() > 0


def test_oracle_sirt_matches_reference(golden, oracle_proj):
    from oracle import solvers as osol
    meta, g = golden
    spec = meta["projector"]["cfg0"]
    n, d, angles = case_geometry(spec)
    w = oracle_proj.build_csr(n, d, angles)
    x_ex = g["cfg0_phantom"]
    x, rec = osol.sirt_solve(w, w @ x_ex, None, 200, x_ex=x_ex)
    assert np.array_equal(x, g["sirt_cfg0_x"])          # bitwise iterate parity
    np.testing.assert_allclose(rec.rel_residual, g["sirt_cfg0_res"], rtol=1e-12)
    np.testing.assert_allclose(rec.rel_err_l2, g["sirt_cfg0_err"], rtol=1e-12)


def test_oracle_bicgstab_within_reference_envelope(golden, oracle_proj):
    """DET_SUM dots vs OpenBLAS ddot: same algorithm, drift at reorder level."""
    from oracle import solvers as osol
    meta, g = golden
    spec = meta["projector"]["w16"]
    n, d, angles = case_geometry(spec)
    w = oracle_proj.build_csr(n, d, angles)
    from paper_1310_0956_b200.phantom import shepp_logan
    ph = shepp_logan(16)
    f = w.T @ (w @ ph)
    x, rec = osol.bicgstab_solve(osol.normal_operator(w, 1.0), f, max_iterations=30)
    ref = g["bicg_w16_res"]
    k = min(len(ref), len(rec.rel_residual))
    np.testing.assert_allclose(rec.rel_residual[:10], ref[:10], rtol=1e-6)
    assert rec.rel_residual[k - 1] < 1e-6 and ref[k - 1] < 1e-6


def test_det_sum_definition():
    from oracle.solvers import det_sum
    rng = np.random.default_rng(0)
    for n in (0, 1, 31, 1024, 1025, 70000, 1_100_000):
        v = rng.standard_normal(n)
        s = det_sum(v)
        assert s == det_sum(v.copy())
        exact = float(np.sum(v.astype(np.longdouble)))
        assert abs(s - exact) <= 1e-12 * max(1.0, np.abs(v).sum())
    # the tree on one chunk: lane sums then s[l] + s[l+16] ... order
    v = np.arange(1024, dtype=np.float64)
    assert det_sum(v) == float(v.sum())


@pytest.mark.parametrize("levels", [2, 3])
def test_oracle_wtg_matches_reference(golden, oracle_proj, levels):
    from oracle import multilevel as oml
    meta, g = golden
    n, d, angles = case_geometry(meta["projector"]["w16"])
    w = oracle_proj.build_csr(n, d, angles)
    root = oml.build_hierarchy(w, 16, 1.0, levels)
    r = g[f"wtg_w16_l{levels}_r"]
    for mult, key in ((False, "hyb"), (True, "mul")):
        got = oml.wtg_apply(root, r, mult)
        assert np.abs(got - g[f"wtg_w16_l{levels}_{key}"]).max() <= 1e-12


JOSEPH = ["jos_tiny_vertical", "jos_tiny_two", "jos_diag8", "jos_miss12", "jos_odd15",
          "jos_w16", "jos_cfg0", "jos_cfg1", "jos_bench160"]


@pytest.mark.parametrize("name", JOSEPH)
def test_oracle_joseph_csr_matches_reference(golden, oracle_proj, name):
    """f4: the oracle's Joseph restatement reproduces the reference's
    build_projector(kernel="joseph") CSR and both products bit for bit."""
    meta, _ = golden
    spec = meta["joseph"][name]
    n, d, angles = case_geometry(spec)
    w = oracle_proj.build_csr(n, d, angles, kernel="joseph")
    assert w.nnz == spec["nnz"]
    assert sha(w.indptr.astype(np.int64)) == spec["indptr"]
    assert sha(w.indices.astype(np.int64)) == spec["indices"]
    assert sha(w.data) == spec["data"]
    x, y = case_vectors(spec, w.shape[0])
    assert sha(oracle_proj.csr_matvec(w, x)) == spec["wx"]
    assert sha(oracle_proj.csr_matvec(w.T.tocsr(), y)) == spec["wty"]   # csc_matvec order
