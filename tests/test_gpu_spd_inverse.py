"""Batched SPD inverse on the fp64 tensor cores (``wmg_spd_inverse``).

The WMG leaves' coarse solves (reference: potrf + cho_solve,
sparse_kernels.py:53-75) use the inverse this kernel computes; it is checked
against float64 LU inverses, against the reference's failure contract
(NotPositiveDefiniteError naming the leading minor potrf would report), and
for the lower-triangle-only input the hierarchy hands it.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _spd(torch, b, p, seed, cond=1e4):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    q, _ = torch.linalg.qr(torch.randn(b, p, p, dtype=torch.float64, device="cuda",
                                       generator=g))
    ev = torch.logspace(0, np.log10(cond), p, dtype=torch.float64, device="cuda")
    a = q @ torch.diag_embed(ev.expand(b, p)) @ q.transpose(1, 2)
    return 0.5 * (a + a.transpose(1, 2))


@pytest.mark.parametrize("p", [128, 256, 640, 100, 300])
def test_spd_inverse_matches_lu(gpu, p):
    torch = gpu
    from paper_1310_0956_b200.sparse_kernels import spd_inverse_
    a = _spd(torch, 3, p, seed=p)
    ref = torch.linalg.inv(a)
    got = a.clone()
    spd_inverse_(got)
    rel = ((got - ref).norm(dim=(1, 2)) / ref.norm(dim=(1, 2))).max().item()
    assert rel <= 1e-10, rel
    # symmetric output, identity residual at kappa * eps
    assert torch.equal(got, got.transpose(1, 2))
    eye = torch.eye(p, dtype=torch.float64, device="cuda")
    assert (a @ got - eye).abs().max().item() <= 1e-9


def test_spd_inverse_reads_lower_triangle_only(gpu):
    torch = gpu
    from paper_1310_0956_b200.sparse_kernels import spd_inverse_
    a = _spd(torch, 2, 384, seed=7)
    full = a.clone()
    low = torch.tril(a)
    low += torch.triu(torch.full_like(a, 1e30), diagonal=1)   # garbage above
    spd_inverse_(full)
    spd_inverse_(low)
    assert torch.equal(full, low)


def test_spd_inverse_single_matrix_and_deterministic(gpu):
    torch = gpu
    from paper_1310_0956_b200.sparse_kernels import spd_inverse_
    a = _spd(torch, 1, 512, seed=3)[0].contiguous()
    x1, x2 = a.clone(), a.clone()
    spd_inverse_(x1)
    spd_inverse_(x2)
    assert torch.equal(x1, x2)
    assert ((x1 - torch.linalg.inv(a)).norm() / x1.norm()).item() <= 1e-10


@pytest.mark.parametrize("bad", [0, 5, 127, 128, 300])
def test_spd_inverse_not_pd_reports_leading_minor(gpu, bad):
    """First failing leading minor, as potrf's info (cholesky_ex) reports it."""
    torch = gpu
    from paper_1310_0956_b200 import NotPositiveDefiniteError
    from paper_1310_0956_b200.sparse_kernels import spd_inverse_
    a = _spd(torch, 3, 384, seed=11, cond=10.0)
    a[1, bad, bad] = -1.0
    _, info = torch.linalg.cholesky_ex(a)
    assert int(info[1]) == bad + 1 and int(info[0]) == 0 and int(info[2]) == 0
    with pytest.raises(NotPositiveDefiniteError, match=f"leaf1: leading minor of order {bad + 1} "):
        spd_inverse_(a.clone(), names=["leaf0", "leaf1", "leaf2"])


def test_hierarchy_leaves_are_inverses_of_the_grams(gpu, golden):
    """Leaf inverse x Galerkin Gram == I on the reference's w40 fixture."""
    torch = gpu
    from conftest import case_geometry
    from paper_1310_0956_b200 import BAND_IDS, build_wmg_hierarchy
    from paper_1310_0956_b200.geometry import Geometry, build_projector
    from paper_1310_0956_b200.multilevel import build_intergrid_set
    meta, _ = golden
    n, d, angles = case_geometry(meta["projector"]["w40"])
    w = build_projector(Geometry(n, d, angles.size, angles=angles))
    lam = 1.0
    h = build_wmg_hierarchy(w, 40, lam, 2)
    wcsr = w.to_scipy()
    grids = build_intergrid_set(40)
    for band in BAND_IDS:
        r = grids[band]
        gram = (r @ (wcsr.T @ wcsr) @ r.T).toarray() + lam * np.eye(400)
        inv = h.root.children[band].coarse_solve.inverse.cpu().numpy()
        np.testing.assert_allclose(inv @ gram, np.eye(400), atol=1e-9)


def test_packed_symmetric_storage_and_symv(gpu):
    """Packed lower-tile storage: lossless round trip; the tile-once symmetric
    GEMV matches the dense product, is deterministic and slices by matrix."""
    torch = gpu
    from paper_1310_0956_b200.sparse_kernels import PackedSymmetric, batched_gemv
    a = _spd(torch, 3, 384, seed=5, cond=1e3)
    pk = PackedSymmetric.pack(a)
    assert pk.data.numel() == 3 * 6 * 128 * 128        # 3 x (3 * 4 / 2) tiles
    assert torch.equal(pk.dense(), a)
    x = torch.randn(3, 384, dtype=torch.float64, device="cuda")
    ref = torch.bmm(a, x.unsqueeze(2)).squeeze(2)
    y1 = batched_gemv(pk, x)
    y2 = batched_gemv(pk, x)
    assert torch.equal(y1, y2)
    assert ((y1 - ref).norm() / ref.norm()).item() <= 1e-14
    y3 = batched_gemv(pk[1:3], x[1:3])
    assert torch.equal(y3, y1[1:3])
    y4 = pk[2].gemv(x[2])
    assert torch.equal(y4, y1[2])


def test_hierarchy_packed_inverses_match_dense(gpu):
    """Leaves of order 256 (n = 64, 3 levels) stored packed: the V-cycle equals
    the dense-inverse cycle to rounding, and WMG-CGLS takes the same path."""
    torch = gpu
    import numpy as np
    from paper_1310_0956_b200 import (SolverConfig, build_geometry, build_projector,
                                      build_wmg_hierarchy, cgls_solve, random_ellipses,
                                      wmg_preconditioner)
    from paper_1310_0956_b200.sparse_kernels import PackedSymmetric
    g = build_geometry(64, 91, 90)
    w = build_projector(g)
    hp = build_wmg_hierarchy(w, 64, 0.0, 3, nu_pre=1, nu_post=1)
    hd = build_wmg_hierarchy(w, 64, 0.0, 3, nu_pre=1, nu_post=1, packed=False)
    assert isinstance(hp.leaf_inverses, PackedSymmetric) and hp.leaf_inverses.p == 256
    assert not isinstance(hd.leaf_inverses, PackedSymmetric)
    assert torch.equal(hp.leaf_inverses.dense(), hd.leaf_inverses)
    v = torch.randn(64 * 64, dtype=torch.float64, device="cuda")
    Mp, Md = wmg_preconditioner(hp), wmg_preconditioner(hd)
    zp, zd = Mp(v), Md(v)
    assert ((zp - zd).norm() / zd.norm()).item() <= 1e-12
    b = w @ random_ellipses(64, 10, seed=0)
    cfg = SolverConfig(max_iterations=30, residual_tolerance=1e-6)
    _, rp = cgls_solve(w, b, precond=Mp, cfg=cfg)
    _, rd = cgls_solve(w, b, precond=Md, cfg=cfg)
    assert rp.iterations[-1] == rd.iterations[-1]
    np.testing.assert_allclose(rp.rel_residual, rd.rel_residual, rtol=1e-8)
