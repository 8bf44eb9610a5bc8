"""Parity of the fp32 projector pair at the sizes the bench measures.

The bench line (``bench.py``) times BASELINE config 3 at n = 4096 (4096 angles,
5793 detectors, float32) through the DEFAULT dispatch: the mirror-packed
symmetric forward ``fwd_sym_kernel`` and the eight-image backprojector
``bwd_sym8_kernel``.  These tests run exactly that dispatch (asserted from the
CUDA kernel names the profiler records) on the bench's own inputs and compare:

* forward rows of >= 8 angles (0, pi/4, pi/2, 3pi/4, ... and the mirror /
  transposition partners) against the pinned CPU oracle
  (``oracle.cproj.forward``, bit-identical to the reference ``W @ x`` of
  /root/reference/pkg/src/wmgtomo/geometry.py:200-206 on exact angle subsets),
  within 1e-5 relative per angle and over the set;
* the full sinogram against the float64 PARITY forward (bit-identical to the
  reference on every golden case), within 1e-5;
* the full backprojection against the float64 parity backprojector
  (geometry.py:209-215), within 1e-5;
* the adjoint identity <W x, y> = <x, W^T y> of the fp32 pair, within 1e-6.

Repeated at n = 2048 (2048 angles, 2897 detectors), the next config-3 size,
which takes the same kernels.
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _kernel_names(torch, fn, want):
    """CUDA kernel names launched by fn() (CUPTI via torch.profiler).  Kernel
    records arrive asynchronously, so fn runs twice per capture and the capture
    is retried if the expected kernel is missing."""
    from torch.profiler import ProfilerActivity, profile
    names = set()
    for _ in range(3):
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            fn()
            fn()
            torch.cuda.synchronize()
        names |= {e.name for e in prof.events() if e.device_type.name == "CUDA"}
        if any(want in k for k in names):
            break
    return names


def _angle_sample(m):
    q = m // 8
    idx = {0, q, 2 * q, 3 * q, 4 * q, 5 * q, 6 * q, 7 * q,     # 0, pi/8, ..., 7pi/8
           1, m - 1, m // 2 - 1, m // 2 + 1, 1025 % m, 3069 % m}
    return np.array(sorted(idx))


@pytest.mark.parametrize("n", [4096, 2048])
def test_default_dispatch_pair_vs_oracle(gpu, oracle_proj, n):
    torch = gpu
    from paper_1310_0956_b200.geometry import build_geometry, build_projector
    m, d = n, int(math.ceil(n * math.sqrt(2.0)))
    g = build_geometry(n, d, m)
    w = build_projector(g, precision="float32")
    assert w.symmetric and w.transposition_closed
    x = np.random.default_rng(3000).uniform(0.0, 1.0, n * n).astype(np.float32)
    y = np.random.default_rng(3001).uniform(0.0, 1.0, m * d).astype(np.float32)
    xd = torch.from_numpy(x).cuda()
    yd = torch.from_numpy(y).cuda()
    sino = torch.empty(m * d, dtype=torch.float32, device="cuda")
    img = torch.empty(n * n, dtype=torch.float32, device="cuda")

    names_f = _kernel_names(torch, lambda: w.forward_(xd, sino), "fwd_sym_kernel")
    names_b = _kernel_names(torch, lambda: w.backward_(yd, img), "bwd_sym8_kernel")
    assert any("fwd_sym_kernel" in k for k in names_f), sorted(names_f)
    assert any("bwd_sym8_kernel" in k for k in names_b), sorted(names_b)

    got_f = sino.double().cpu().numpy().reshape(m, d)
    got_b = img.double().cpu().numpy()
    x64, y64 = x.astype(np.float64), y.astype(np.float64)

    # (1) forward rows of sampled angles vs the oracle (exact reference rows)
    idx = _angle_sample(m)
    assert {0, m // 4, m // 2, 3 * m // 4} <= set(idx.tolist())
    ref_rows = oracle_proj.forward(n, d, g.angles[idx], x64).reshape(idx.size, d)
    for k, a in enumerate(idx):
        r = ref_rows[k]
        assert np.linalg.norm(got_f[a] - r) <= 1e-5 * np.linalg.norm(r), int(a)
    assert np.linalg.norm(got_f[idx] - ref_rows) <= 1e-5 * np.linalg.norm(ref_rows)

    # (2) full sinogram and (3) full backprojection vs the float64 parity kernels
    wp = build_projector(g)
    ref_f = wp.forward(torch.from_numpy(x64).cuda()).cpu().numpy().reshape(m, d)
    assert np.array_equal(ref_f[idx], ref_rows)          # parity kernel == oracle rows
    assert np.linalg.norm(got_f - ref_f) <= 1e-5 * np.linalg.norm(ref_f)
    ref_b = wp.backward(torch.from_numpy(y64).cuda()).cpu().numpy()
    assert np.linalg.norm(got_b - ref_b) <= 1e-5 * np.linalg.norm(ref_b)

    # (4) adjoint identity of the fp32 pair
    lhs = float(np.dot(got_f.ravel(), y64))
    rhs = float(np.dot(x64, got_b))
    assert abs(lhs - rhs) <= 1e-6 * abs(lhs)


@pytest.mark.parametrize("n,m,seg,stride", [(1280, 720, 8, 1), (1536, 1000, 8, 1),
                                            (1152, 600, 8, 1), (1024, 1024, 8, 1),
                                            (1792, 896, 8, 1), (1920, 1920, 1, 4)])
def test_forward_block_layouts_vs_parity(gpu, n, m, seg, stride):
    """The symmetric forward's block layouts around their switch (below n = 1792,
    and for launches of fewer than 8000 four-octet blocks, one ray octet per block
    with the slab range in 8 row segments; else four ray octets 4 apart per
    block, unsplit), on angle counts that are not
    multiples of the 4-angle groups' super-blocks: the full sinogram within
    1e-5 of the float64 parity forward (reference geometry.py:200-206), every row
    within 1e-5, the layout asserted from the launched kernel's template."""
    torch = gpu
    from paper_1310_0956_b200.geometry import build_geometry, build_projector
    d = int(math.ceil(n * math.sqrt(2.0)))
    g = build_geometry(n, d, m)
    w = build_projector(g, precision="float32")
    x = np.random.default_rng(n + m).uniform(0.0, 1.0, n * n).astype(np.float32)
    xd = torch.from_numpy(x).cuda()
    sino = torch.empty(m * d, dtype=torch.float32, device="cuda")
    names = _kernel_names(torch, lambda: w.forward_(xd, sino), "fwd_sym_kernel")
    k = [s for s in names if "fwd_sym_kernel" in s]
    assert k and all(s.split("(")[0].replace(" ", "").endswith(f",{seg},{stride}>") for s in k), k
    got = sino.double().cpu().numpy().reshape(m, d)
    ref = build_projector(g).forward(torch.from_numpy(x.astype(np.float64)).cuda())
    ref = ref.cpu().numpy().reshape(m, d)
    assert np.linalg.norm(got - ref) <= 1e-5 * np.linalg.norm(ref)
    err = np.linalg.norm(got - ref, axis=1)
    nrm = np.linalg.norm(ref, axis=1)
    assert np.all(err <= 1e-5 * np.maximum(nrm, 1e-30)), int(np.argmax(err / np.maximum(nrm, 1e-30)))


@pytest.mark.parametrize("n,m,passes", [(3072, 1024, 3), (4096, 128, 4), (3072, 128, 1)])
def test_banded_forward_passes_vs_parity(gpu, n, m, passes):
    """When the padded planes exceed the L2 the forward runs as slab-band passes
    that add their partial ray sums (projector_fast.cu, fwd_v2_impl): the
    unsplit form from 128 MB of planes (n = 3072: 3 passes), the 8-segment form
    that few angles (a rank's shard) take from 200 MB (n = 4096: 4 passes; one
    launch at n = 3072).  The pass count is asserted from the launches, the
    sinogram checked against the float64 parity forward (reference
    geometry.py:200-206) within 1e-5 per row."""
    torch = gpu
    from torch.profiler import ProfilerActivity, profile
    from paper_1310_0956_b200.geometry import build_geometry, build_projector
    d = int(math.ceil(n * math.sqrt(2.0)))
    g = build_geometry(n, d, m)
    w = build_projector(g, precision="float32")
    x = np.random.default_rng(n).uniform(0.0, 1.0, n * n).astype(np.float32)
    xd = torch.from_numpy(x).cuda()
    sino = torch.empty(m * d, dtype=torch.float32, device="cuda")
    w.forward_(xd, sino)
    torch.cuda.synchronize()
    count = 0
    for _ in range(3):
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            w.forward_(xd, sino)
            torch.cuda.synchronize()
        count = sum(1 for e in prof.events()
                    if e.device_type.name == "CUDA" and "fwd_sym_kernel" in e.name)
        if count:
            break
    assert count == passes, count
    got = sino.double().cpu().numpy().reshape(m, d)
    ref = build_projector(g).forward(torch.from_numpy(x.astype(np.float64)).cuda())
    ref = ref.cpu().numpy().reshape(m, d)
    err = np.linalg.norm(got - ref, axis=1)
    nrm = np.linalg.norm(ref, axis=1)
    assert np.all(err <= 1e-5 * np.maximum(nrm, 1e-30))


@pytest.mark.parametrize("n,m,eight", [(1728, 432, True), (1664, 416, False)])
def test_eight_image_backprojector_threshold_vs_parity(gpu, n, m, eight):
    """The eight-image backprojector takes over from 370 quadrant tile pairs
    (n = 1728; the four-image run layout below): on both sides of the switch
    the backprojection (and the banded form where it exists) is within 1e-5 of
    the float64 parity backprojector (reference geometry.py:209-215) and the
    kernel is the expected one."""
    torch = gpu
    from paper_1310_0956_b200.geometry import build_geometry, build_projector
    d = int(math.ceil(n * math.sqrt(2.0)))
    g = build_geometry(n, d, m)
    w = build_projector(g, precision="float32")
    y = np.random.default_rng(n).uniform(0.0, 1.0, m * d).astype(np.float32)
    yd = torch.from_numpy(y).cuda()
    img = torch.empty(n * n, dtype=torch.float32, device="cuda")
    want = "bwd_sym8_kernel" if eight else "bwd_symrun_kernel"
    names = _kernel_names(torch, lambda: w.backward_(yd, img), want)
    assert any(want in k for k in names), sorted(names)
    assert (w.backward_bands() > 0) == eight
    ref = build_projector(g).backward(torch.from_numpy(y.astype(np.float64)).cuda())
    ref = ref.cpu().numpy()
    got = img.double().cpu().numpy()
    assert np.linalg.norm(got - ref) <= 1e-5 * np.linalg.norm(ref)
    assert np.max(np.abs(got - ref)) <= 1e-4 * np.max(np.abs(ref))
    if eight:
        qt = w.backward_bands()
        out = torch.full_like(img, float("nan"))
        for s0, s1 in ((0, 7), (7, qt // 2), (qt // 2, qt)):
            w.backward_band_(yd, out, s0, s1)
        assert torch.equal(out, img)


def test_prefer_concurrent_forward_form(gpu):
    """``prefer_concurrent`` keeps a few-block forward launch (here n = 2048 with
    128 angles) in the unsplit four-octet form instead of the 8-segment form:
    different kernels, the same sinogram to fp32 rounding."""
    torch = gpu
    from paper_1310_0956_b200.geometry import build_geometry, build_projector
    n, m = 2048, 128
    d = int(math.ceil(n * math.sqrt(2.0)))
    g = build_geometry(n, d, m)
    x = torch.rand(n * n, device="cuda", generator=torch.Generator("cuda").manual_seed(7))
    out = {}
    for conc in (False, True):
        w = build_projector(g, precision="float32")
        assert w.prefer_concurrent(conc)
        s = torch.empty(m * d, device="cuda")
        names = _kernel_names(torch, lambda: w.forward_(x, s), "fwd_sym_kernel")
        k = [q.split("(")[0].replace(" ", "") for q in names if "fwd_sym_kernel" in q]
        assert k and all(q.endswith(",1,4>" if conc else ",8,1>") for q in k), k
        out[conc] = s
    rel = float((out[True] - out[False]).norm() / out[False].norm())
    assert rel <= 1e-6, rel


def test_pdl_chained_passes_in_a_captured_iteration(gpu):
    """The banded forward's passes are chained with programmatic dependent
    launches (pass b + 1 starts while pass b drains and waits for it before it
    adds its partial sums).  Inside a captured CGLS iteration (stream capture
    turns the attribute into programmatic graph edges) the solve must equal the
    eager one bit for bit, and repeated forwards must agree bit for bit."""
    torch = gpu
    from paper_1310_0956_b200 import SolverConfig, cgls_solve
    from paper_1310_0956_b200.geometry import build_geometry, build_projector
    n, m = 3584, 64                      # 213 MB of planes: 4 passes of the 8-segment form
    d = int(math.ceil(n * math.sqrt(2.0)))
    g = build_geometry(n, d, m)
    w = build_projector(g, precision="float32")
    x = torch.rand(n * n, device="cuda", generator=torch.Generator("cuda").manual_seed(11))
    s1 = torch.empty(m * d, device="cuda")
    s2 = torch.empty(m * d, device="cuda")
    count = 0
    from torch.profiler import ProfilerActivity, profile
    for _ in range(3):
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            w.forward_(x, s1)
            torch.cuda.synchronize()
        count = sum(1 for e in prof.events()
                    if e.device_type.name == "CUDA" and "fwd_sym_kernel" in e.name)
        if count:
            break
    assert count == 4, count
    for _ in range(3):
        w.forward_(x, s2)
        assert torch.equal(s1, s2)
    ref = build_projector(g).forward(x.double())
    assert float((s1.double() - ref).norm() / ref.norm()) <= 1e-5
    b = s1.double()
    cfg = SolverConfig(max_iterations=4, residual_tolerance=0.0)
    xg, rg = cgls_solve(w, b, cfg=cfg)                 # iterations 2.. replay a captured graph
    xe, re_ = cgls_solve(w, b, cfg=cfg, graph=False)
    assert torch.equal(xg, xe)
    assert rg.rel_residual == re_.rel_residual
