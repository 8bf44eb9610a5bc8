"""Projector parity on the B200 (calls go through the C ABI via ctypes).

* PARITY mode (float64): the GPU-exported CSR, W x, W^T y, row and column sums
  are BIT-IDENTICAL to the reference (sha256 of the frozen reference results)
  on every golden case, including exact angle subsets of config 3 at n = 4096.
* FAST mode: float32 data within 1e-5 relative (north_star), float64 fast
  within 1e-12 relative, against the pinned CPU oracle.
"""
import hashlib

import numpy as np
import pytest

from conftest import case_geometry, case_vectors

pytestmark = pytest.mark.gpu


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


CASES = ["tiny_vertical", "tiny_two", "diag8", "miss12", "w16", "w40", "cfg0", "cfg1",
         "bench160", "cfg3_512_sub", "cfg3_1024_sub", "cfg3_2048_sub", "cfg3_4096_sub"]


def _proj(spec, **kw):
    from paper_1310_0956_b200.geometry import Geometry, build_projector
    n, d, angles = case_geometry(spec)
    return build_projector(Geometry(n, d, angles.size, angles=angles), **kw)


@pytest.mark.parametrize("name", CASES)
def test_parity_bitwise_vs_reference(gpu, golden, name):
    torch = gpu
    meta, _ = golden
    spec = meta["projector"][name]
    w = _proj(spec)
    x, y = case_vectors(spec, w.shape[0])
    xd = torch.from_numpy(x).cuda()
    yd = torch.from_numpy(y).cuda()
    anomaly = torch.zeros(1, dtype=torch.int32, device="cuda")
    wx = torch.empty(w.shape[0], dtype=torch.float64, device="cuda")
    wty = torch.empty(w.shape[1], dtype=torch.float64, device="cuda")
    w.forward_(xd, wx, anomaly=anomaly)
    w.backward_(yd, wty, anomaly=anomaly)
    torch.cuda.synchronize()
    assert int(anomaly.item()) == 0
    assert sha(wx.cpu().numpy()) == spec["wx"]
    assert sha(wty.cpu().numpy()) == spec["wty"]
    assert sha(w.row_sums_dev().cpu().numpy()) == spec["rows"]
    assert sha(w.col_sums_dev().cpu().numpy()) == spec["cols"]


@pytest.mark.parametrize("name", ["tiny_vertical", "tiny_two", "diag8", "miss12", "w16",
                                  "w40", "cfg0", "cfg1", "cfg3_1024_sub"])
def test_gpu_csr_entry_for_entry(gpu, golden, name):
    meta, _ = golden
    spec = meta["projector"][name]
    w = _proj(spec)
    indptr, cols, vals, anomaly = w.csr_device()
    assert anomaly == 0
    assert int(indptr[-1]) == spec["nnz"]
    assert sha(indptr.cpu().numpy()) == spec["indptr"]
    assert sha(cols.cpu().numpy()) == spec["indices"]
    assert sha(vals.cpu().numpy()) == spec["data"]


@pytest.mark.parametrize("name", ["w16", "w40", "cfg0", "cfg1", "bench160", "cfg3_512_sub",
                                  "cfg3_1024_sub", "cfg3_2048_sub", "cfg3_4096_sub"])
def test_fast_fp32_within_1e5(gpu, golden, oracle_proj, name):
    torch = gpu
    meta, _ = golden
    spec = meta["projector"][name]
    n, d, angles = case_geometry(spec)
    w = _proj(spec, precision="float32")
    rs = np.random.default_rng(123)
    x = rs.uniform(0.0, 1.0, n * n)
    y = rs.uniform(0.0, 1.0, w.shape[0])
    ref_f = oracle_proj.forward(n, d, angles, x)
    ref_b = oracle_proj.backward(n, d, angles, y) if n <= 1024 else None
    got_f = w.forward(torch.from_numpy(x.astype(np.float32)).cuda()).double().cpu().numpy()
    assert np.linalg.norm(got_f - ref_f) <= 1e-5 * np.linalg.norm(ref_f)
    got_b = w.backward(torch.from_numpy(y.astype(np.float32)).cuda()).double().cpu().numpy()
    if ref_b is None:
        # n >= 2048: W^T y against the parity kernel (bit-identical to the reference)
        wp = _proj(spec)
        ref_b = wp.backward(torch.from_numpy(y).cuda()).cpu().numpy()
    assert np.linalg.norm(got_b - ref_b) <= 1e-5 * np.linalg.norm(ref_b)


@pytest.mark.parametrize("name", ["w40", "cfg0", "cfg1", "cfg3_1024_sub"])
def test_fast_fp64_within_1e12(gpu, golden, name):
    torch = gpu
    meta, _ = golden
    spec = meta["projector"][name]
    wp = _proj(spec)
    wf = _proj(spec, precision="float64", mode="fast")
    x, y = case_vectors(spec, wp.shape[0])
    xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    for a, b in ((wf.forward(xd), wp.forward(xd)), (wf.backward(yd), wp.backward(yd))):
        a, b = a.cpu().numpy(), b.cpu().numpy()
        assert np.linalg.norm(a - b) <= 1e-12 * np.linalg.norm(b)


def test_numpy_roundtrip_and_protocol(gpu, golden):
    meta, g = golden
    spec = meta["projector"]["w16"]
    w = _proj(spec)
    x, y = case_vectors(spec, w.shape[0])
    assert isinstance(w @ x, np.ndarray)
    assert sha(w @ x) == spec["wx"]
    assert sha(w.T @ y) == spec["wty"]
    assert sha(w.T.tocsr() @ y) == spec["wty"]
    assert w.tocsr() is w and w.shape == (24 * 24, 256)


def test_adjoint_identity_fast(gpu):
    torch = gpu
    from paper_1310_0956_b200.geometry import build_geometry, build_projector
    w = build_projector(build_geometry(300, 425, 301), precision="float32")
    rs = np.random.default_rng(5)
    x = torch.from_numpy(rs.standard_normal(w.shape[1])).cuda()
    y = torch.from_numpy(rs.standard_normal(w.shape[0])).cuda()
    wf = build_projector(build_geometry(300, 425, 301), precision="float64", mode="fast")
    wx = wf.forward(x)
    lhs = float(wx.dot(y))
    rhs = float(x.dot(wf.backward(y)))
    # forward (slab walk) and backward (pixel trapezoid) are independent
    # evaluations of the same weights: adjoint to rounding
    assert abs(lhs - rhs) <= 1e-13 * float(wx.norm() * y.norm())


def test_dimension_checks(gpu):
    from paper_1310_0956_b200 import DimensionMismatchError, apply, apply_transpose
    from paper_1310_0956_b200.geometry import build_geometry, build_projector
    w = build_projector(build_geometry(16, 24, 24))
    with pytest.raises(DimensionMismatchError):
        apply(w, np.ones(7))
    with pytest.raises(DimensionMismatchError):
        apply_transpose(w, np.ones(7))


@pytest.mark.parametrize("mode", ["force", "tma", "bwd8x4", "bwdrun32", "bwdrun64", "bwdsym8",
                                  "bwdrun"])
@pytest.mark.parametrize("n,d,m", [(256, 363, 180), (512, 725, 512), (320, 453, 64)])
def test_symmetric_fast_paths(gpu, oracle_proj, n, d, m, mode):
    """Full equiangular grids take the mirror-symmetric kernels: same result as
    the plain fast kernels (1e-6) and within 1e-5 of the float64 reference.
    Modes: the default kernels; the TMA forward; the backprojector's 8x4-block
    float4-window layout and its run layout with 4 / 8 rows per thread (the
    64-row tiles are the n = 4096 default; n = 320 falls back to 32 rows); the
    eight-image (transposition) backprojector forced at these sizes, and
    disabled (m = 180, 512 and 64 are multiples of 4: transposition-closed)."""
    torch = gpu
    from paper_1310_0956_b200.geometry import build_geometry, build_projector
    g = build_geometry(n, d, m)
    w = build_projector(g, precision="float32")
    assert w.symmetric
    assert w.set_symmetry(mode)
    rs = np.random.default_rng(n)
    x = rs.uniform(0.0, 1.0, n * n)
    y = rs.uniform(0.0, 1.0, m * d)
    xd = torch.from_numpy(x.astype(np.float32)).cuda()
    yd = torch.from_numpy(y.astype(np.float32)).cuda()
    fs, bs = w.forward(xd).double(), w.backward(yd).double()
    assert not w.set_symmetry(False)
    fp, bp = w.forward(xd).double(), w.backward(yd).double()
    assert w.set_symmetry(mode)
    assert float((fs - fp).norm()) <= 1e-6 * float(fp.norm())
    assert float((bs - bp).norm()) <= 1e-6 * float(bp.norm())
    ref_f = oracle_proj.forward(n, d, g.angles, x)
    ref_b = oracle_proj.backward(n, d, g.angles, y)
    assert np.linalg.norm(fs.cpu().numpy() - ref_f) <= 1e-5 * np.linalg.norm(ref_f)
    assert np.linalg.norm(bs.cpu().numpy() - ref_b) <= 1e-5 * np.linalg.norm(ref_b)


def test_symmetry_not_used_for_asymmetric_sets(gpu):
    from paper_1310_0956_b200.geometry import Geometry, build_geometry, build_projector
    assert not build_projector(build_geometry(100, 145, 64), precision="float32").symmetric
    # odd m: pi/2 is missing, the mirror pairs (k, m - k) and the axis angle 0 remain
    assert build_projector(build_geometry(128, 181, 63), precision="float32").symmetric
    a = np.sort(np.random.default_rng(0).uniform(0, np.pi, 64))
    assert not build_projector(Geometry(128, 181, 64, angles=a), precision="float32").symmetric


@pytest.mark.parametrize("n,d,m", [(256, 363, 180), (512, 725, 512)])
def test_symmetric_fast_fp64(gpu, n, d, m):
    """float64 symmetric kernels (forced) against the bit-exact parity kernels."""
    torch = gpu
    from paper_1310_0956_b200.geometry import build_geometry, build_projector
    g = build_geometry(n, d, m)
    wp = build_projector(g)
    wf = build_projector(g, precision="float64", mode="fast")
    assert wf.set_symmetry("force")
    rs = np.random.default_rng(n + 1)
    x = torch.from_numpy(rs.uniform(0.0, 1.0, n * n)).cuda()
    y = torch.from_numpy(rs.uniform(0.0, 1.0, m * d)).cuda()
    for a, b in ((wf.forward(x), wp.forward(x)), (wf.backward(y), wp.backward(y))):
        assert float((a - b).norm()) <= 1e-12 * float(b.norm())


def test_symmetric_fast_n1024_default_dispatch(gpu):
    """At n = 1024 the default dispatch takes the symmetric kernels; compare with
    the parity kernels (bit-identical to the reference)."""
    torch = gpu
    from paper_1310_0956_b200.geometry import build_geometry, build_projector
    n, d, m = 1024, 1449, 1024
    g = build_geometry(n, d, m)
    wp = build_projector(g)
    wf = build_projector(g, precision="float32")
    rs = np.random.default_rng(7)
    x = rs.uniform(0.0, 1.0, n * n)
    y = rs.uniform(0.0, 1.0, m * d)
    ff = wf.forward(torch.from_numpy(x.astype(np.float32)).cuda()).double()
    bb = wf.backward(torch.from_numpy(y.astype(np.float32)).cuda()).double()
    fr = wp.forward(torch.from_numpy(x).cuda())
    br = wp.backward(torch.from_numpy(y).cuda())
    assert float((ff - fr).norm()) <= 1e-5 * float(fr.norm())
    assert float((bb - br).norm()) <= 1e-5 * float(br.norm())


@pytest.mark.parametrize("n,d,m,world", [(256, 363, 180, 2), (256, 363, 180, 4),
                                         (256, 363, 180, 8), (128, 181, 63, 3),
                                         (1024, 1449, 720, 8)])
def test_symmetric_kernels_on_mirror_shards(gpu, oracle_proj, n, d, m, world):
    """Per-rank angle shards of sharding.shard_angles(..., "mirror") are closed
    under theta -> pi - theta; most hold neither axis angle.  They keep the
    symmetric kernels (table-driven mirror pairs) and stay within 1e-5 of the
    float64 reference rows of those angles."""
    torch = gpu
    from paper_1310_0956_b200.geometry import build_geometry, build_projector
    from paper_1310_0956_b200.sharding import shard_angles
    g = build_geometry(n, d, m)
    rs = np.random.default_rng(n + m + world)
    x = rs.uniform(0.0, 1.0, n * n)
    xd = torch.from_numpy(x.astype(np.float32)).cuda()
    for rank in range(world):
        idx = shard_angles(m, world, rank, "mirror")
        sub = g.subset(idx)
        w = build_projector(sub, precision="float32")
        assert w.symmetric and w.set_symmetry("force")
        y = rs.uniform(0.0, 1.0, idx.size * d)
        ref_f = oracle_proj.forward(n, d, sub.angles, x)
        ref_b = oracle_proj.backward(n, d, sub.angles, y)
        got_f = w.forward(xd).double().cpu().numpy()
        got_b = w.backward(torch.from_numpy(y.astype(np.float32)).cuda()).double().cpu().numpy()
        assert np.linalg.norm(got_f - ref_f) <= 1e-5 * np.linalg.norm(ref_f), rank
        assert np.linalg.norm(got_b - ref_b) <= 1e-5 * np.linalg.norm(ref_b), rank
        if n >= 1024:
            wd = build_projector(sub, precision="float64", mode="fast")
            assert wd.set_symmetry("force")
            f64 = wd.forward(torch.from_numpy(x).cuda()).cpu().numpy()
            assert np.linalg.norm(f64 - ref_f) <= 1e-12 * np.linalg.norm(ref_f), rank


@pytest.mark.parametrize("n,d,m,world", [(256, 363, 180, 2), (256, 363, 180, 8),
                                         (512, 725, 512, 4), (1024, 1449, 720, 8)])
def test_eight_image_backprojector_on_quad_shards(gpu, oracle_proj, n, d, m, world):
    """Shards of the "quad" scheme are mirror- and transposition-closed: the
    eight-image backprojector (forced) stays within 1e-5 of the float64
    reference rows of the shard's angles, like the four-image run layout."""
    torch = gpu
    from paper_1310_0956_b200.geometry import build_geometry, build_projector
    from paper_1310_0956_b200.sharding import shard_angles
    g = build_geometry(n, d, m)
    rs = np.random.default_rng(7 * n + world)
    for rank in range(world):
        idx = shard_angles(m, world, rank, "quad")
        sub = g.subset(idx)
        w = build_projector(sub, precision="float32")
        assert w.symmetric and w.transposition_closed
        y = rs.uniform(0.0, 1.0, idx.size * d)
        yd = torch.from_numpy(y.astype(np.float32)).cuda()
        ref_b = oracle_proj.backward(n, d, sub.angles, y)
        for mode in ("bwdsym8", "bwdrun"):
            assert w.set_symmetry(mode)
            got = w.backward(yd).double().cpu().numpy()
            assert np.linalg.norm(got - ref_b) <= 1e-5 * np.linalg.norm(ref_b), (rank, mode)
    # a mirror shard need not be transposition-closed (m = 180, 4 ranks: rank 0
    # holds theta_4 but not theta_86 = pi/2 - theta_4); then the run layout runs
    if m == 180:
        wm = build_projector(g.subset(shard_angles(m, 4, 0, "mirror")), precision="float32")
        assert wm.symmetric and not wm.transposition_closed


@pytest.mark.parametrize("mode", ["bwdsym8", "bwdrun", "bwdrun64"])
def test_fp32_backprojector_float64_vectors_and_accumulate(gpu, oracle_proj, mode):
    """fp32 arithmetic on float64 vectors (configs 2 and 4: float64 Krylov
    vectors) and x += W^T y, through each symmetric backprojector layout."""
    torch = gpu
    from paper_1310_0956_b200.geometry import build_geometry, build_projector
    n, d, m = 256, 363, 180
    g = build_geometry(n, d, m)
    w = build_projector(g, precision="float32")
    assert w.set_symmetry(mode)
    rs = np.random.default_rng(17)
    y = rs.uniform(-1.0, 1.0, m * d)
    x0 = rs.uniform(-1.0, 1.0, n * n)
    ref = oracle_proj.backward(n, d, g.angles, y)
    yd = torch.from_numpy(y).cuda()
    out = torch.empty(n * n, dtype=torch.float64, device="cuda")
    w.backward_(yd, out)
    assert np.linalg.norm(out.cpu().numpy() - ref) <= 1e-5 * np.linalg.norm(ref)
    acc = torch.from_numpy(x0).cuda()
    w.backward_(yd, acc, accumulate=True)
    assert np.linalg.norm(acc.cpu().numpy() - (x0 + ref)) <= 1e-5 * np.linalg.norm(x0 + ref)


@pytest.mark.parametrize("n,d,m", [(1, 1, 1), (2, 3, 2), (3, 5, 3), (17, 9, 7), (64, 91, 8),
                                   (64, 30, 2), (100, 147, 12), (128, 181, 4), (128, 50, 16)])
@pytest.mark.parametrize("precision", ["float32", "float64"])
def test_fast_paths_edge_geometries(gpu, oracle_proj, n, d, m, precision):
    """Tiny / odd grids, few detectors (rays missing the grid), few angles,
    equiangular and random angle sets: the fast kernels stay within their
    tolerance of the exact reference weights (and never read out of bounds)."""
    torch = gpu
    from paper_1310_0956_b200.geometry import Geometry, build_geometry, build_projector
    rs = np.random.default_rng(n * 131 + d * 7 + m)
    geoms = [build_geometry(n, d, m)]
    if m > 1:
        geoms.append(Geometry(n, d, m, angles=np.sort(rs.uniform(0.0, np.pi, m))))
    tol = 1e-5 if precision == "float32" else 1e-12
    dt = torch.float32 if precision == "float32" else torch.float64
    for g in geoms:
        w = build_projector(g, precision=precision, mode="fast")
        x = rs.uniform(0.0, 1.0, n * n)
        y = rs.uniform(0.0, 1.0, m * d)
        ref_f = oracle_proj.forward(n, d, g.angles, x)
        ref_b = oracle_proj.backward(n, d, g.angles, y)
        for sym in (True, "force", False):
            w.set_symmetry(sym)
            f = w.forward(torch.from_numpy(x).to(dt).cuda()).double().cpu().numpy()
            b = w.backward(torch.from_numpy(y).to(dt).cuda()).double().cpu().numpy()
            assert np.linalg.norm(f - ref_f) <= tol * max(np.linalg.norm(ref_f), 1e-30) + 1e-30
            assert np.linalg.norm(b - ref_b) <= tol * max(np.linalg.norm(ref_b), 1e-30) + 1e-30


@pytest.mark.parametrize("n,d,m,precision", [(256, 363, 180, "float64"), (256, 363, 180, "float32"),
                                             (1024, 1449, 64, "float32"), (100, 147, 12, "float64")])
def test_batched_pair_matches_single_calls(gpu, n, d, m, precision):
    """wmg_forward_batch / wmg_backward_batch give each item bit-identically
    what the single-image calls give (batch 0 is a no-op)."""
    torch = gpu
    from paper_1310_0956_b200.geometry import build_geometry, build_projector
    w = build_projector(build_geometry(n, d, m), precision=precision, mode="fast")
    dt = torch.float32 if precision == "float32" else torch.float64
    X = torch.rand(3, n * n, dtype=dt, device="cuda")
    Y = torch.rand(3, m * d, dtype=dt, device="cuda")
    SF = torch.empty(3, m * d, dtype=dt, device="cuda")
    SB = torch.empty(3, n * n, dtype=dt, device="cuda")
    w.forward_batch_(X, SF)
    w.backward_batch_(Y, SB)
    for b in range(3):
        f = torch.empty(m * d, dtype=dt, device="cuda")
        o = torch.empty(n * n, dtype=dt, device="cuda")
        w.forward_(X[b], f)
        w.backward_(Y[b], o)
        assert torch.equal(f, SF[b]) and torch.equal(o, SB[b])
    w.forward_batch_(X[:0], SF[:0])
    w.backward_batch_(Y[:0], SB[:0])
