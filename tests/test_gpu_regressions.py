"""Regression tests for defects found in review."""
import threading

import numpy as np
import pytest


@pytest.mark.gpu
def test_graphed_cgls_recovers_after_breakdown(gpu):
    """A breakdown (NaN right-hand side) must not leave the cached graphed
    CGLS context's breakdown flag set for later solves on the same projector."""
    from paper_1310_0956_b200 import SolverConfig, build_geometry, build_projector, cgls_solve
    g = build_geometry(64, 91, 90)
    w = build_projector(g)
    x = np.random.default_rng(0).uniform(0.0, 1.0, 64 * 64)
    b = w @ x
    cfg = SolverConfig(max_iterations=30)
    _, rec_ok = cgls_solve(w, b, cfg=cfg)
    bad = b.copy()
    bad[45 * 91 + 45] = np.nan          # the central ray of angle 45 (edge rays miss the grid)
    _, rec_bad = cgls_solve(w, bad, cfg=cfg)
    assert rec_bad.status == "breakdown"
    _, rec = cgls_solve(w, b, cfg=cfg)
    assert rec.status == "max-iterations" and rec.iterations[-1] == 30
    assert rec.rel_residual == rec_ok.rel_residual


@pytest.mark.gpu
def test_fp64_forward_after_symmetry_switch(gpu):
    """The generic float64 forward stores an unpadded transposed image in the
    workspace the padded symmetric path reads; switching to the symmetric
    kernels afterwards must not read stale margins."""
    torch = gpu
    from paper_1310_0956_b200.geometry import build_geometry, build_projector
    n, d, m = 1024, 1449, 180
    g = build_geometry(n, d, m)
    wp = build_projector(g)
    wf = build_projector(g, precision="float64", mode="fast")
    x = torch.from_numpy(np.random.default_rng(1).uniform(0.0, 1.0, n * n)).cuda()
    ref = wp.forward(x)
    a = wf.forward(x)                       # auto: generic path at this size
    assert float((a - ref).norm()) <= 1e-12 * float(ref.norm())
    assert wf.set_symmetry("force")
    b = wf.forward(x)                       # padded symmetric planes, same workspace
    assert float((b - ref).norm()) <= 1e-12 * float(ref.norm())
    wf.set_symmetry(False)
    c = wf.forward(x)
    assert float((c - ref).norm()) <= 1e-12 * float(ref.norm())


@pytest.mark.gpu
def test_concurrent_spd_inverses_from_two_threads(gpu):
    """wmg_spd_inverse shares its look-ahead stream and events per device: two
    host threads inverting on their own streams must both get correct inverses."""
    torch = gpu
    from paper_1310_0956_b200.sparse_kernels import spd_inverse_
    p = 512
    rs = np.random.default_rng(3)
    mats = []
    for _ in range(2):
        a = rs.standard_normal((p, p))
        mats.append(a @ a.T + p * np.eye(p))
    outs = [None, None]
    errs = []

    def run(i):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                G = torch.from_numpy(np.stack([mats[i]] * 3)).cuda()
                for _ in range(5):
                    H = G.clone()
                    spd_inverse_(H)
                st.synchronize()
                outs[i] = H.cpu().numpy()
        except Exception as exc:   # pragma: no cover
            errs.append(exc)

    th = [threading.Thread(target=run, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for i in range(2):
        ref = np.linalg.inv(mats[i])
        for b in range(3):
            assert np.linalg.norm(outs[i][b] - ref) <= 1e-10 * np.linalg.norm(ref)


def test_graph_capture_gc_pause_is_reference_counted():
    from paper_1310_0956_b200 import _device as D
    import gc
    was = gc.isenabled()
    gc.enable()
    try:
        D._gc_pause()
        D._gc_pause()
        D._gc_resume()
        assert not gc.isenabled()          # the outer capture is still running
        D._gc_resume()
        assert gc.isenabled()
    finally:
        if not was:
            gc.disable()
