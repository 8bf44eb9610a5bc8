"""Staged host -> device copies of numpy vectors (wmg_h2d_staged, csrc/hostio.cu):
the path every numpy `w @ x` / `w.T @ y` call (geometry.py:200-215 semantics)
takes for vectors of 64 KB and more."""
import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_1310_0956_b200 import _device as D  # noqa: E402
from paper_1310_0956_b200 import _native as N  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("nbytes", [65536, (4 << 20) - 4, 4 << 20, (9 << 20) + 12, 37 << 20])
@pytest.mark.parametrize("threads", [1, 3, 8])
def test_staged_h2d_matches_source(nbytes, threads):
    rng = np.random.default_rng(nbytes + threads)
    a = rng.standard_normal(nbytes // 4).astype(np.float32)
    old = D._STAGE_THREADS
    D._STAGE_THREADS = threads
    try:
        out = D._h2d_staged(a, torch.float32, torch.device("cuda", 0))
        torch.cuda.synchronize()
    finally:
        D._STAGE_THREADS = old
    assert np.array_equal(out.cpu().numpy(), a)


def test_staged_h2d_validation():
    t = torch.empty(4, device="cuda")
    buf = torch.empty(16, dtype=torch.uint8).pin_memory()
    a = np.zeros(4, np.float32)
    with pytest.raises(ValueError):
        N.call("wmg_h2d_staged", t.data_ptr(), a.ctypes.data, 16, buf.data_ptr(), 0, 0)
    with pytest.raises(ValueError):
        N.call("wmg_h2d_staged", t.data_ptr(), None, 16, buf.data_ptr(), 4, 0)
    N.call("wmg_h2d_staged", t.data_ptr(), a.ctypes.data, 0, buf.data_ptr(), 4, 0)   # no-op


def test_concurrent_numpy_calls_from_threads():
    """Two host threads streaming numpy pairs through one projector each: the
    shared copy pool serialises the staged copies, results stay exact."""
    from paper_1310_0956_b200 import build_geometry, build_projector
    n = 512
    g = build_geometry(n, 725, 64)
    outs, errs = {}, []

    def work(k):
        try:
            torch.cuda.set_device(0)
            w = build_projector(g, precision="float32")
            rng = np.random.default_rng(k)
            x = rng.random(n * n, dtype=np.float32)
            y = rng.random(w.shape[0], dtype=np.float32)
            ref_s = w.forward(torch.from_numpy(x).cuda()).cpu().numpy()
            ref_i = w.backward(torch.from_numpy(y).cuda()).cpu().numpy()
            for _ in range(20):
                s = w @ x
                i = w.T @ y
                outs[k] = (np.array_equal(s, ref_s), np.array_equal(i, ref_i))
        except Exception as e:   # pragma: no cover - reported below
            errs.append(e)

    th = [threading.Thread(target=work, args=(k,)) for k in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    assert outs == {0: (True, True), 1: (True, True)}


def test_pinned_numpy_result_fed_back():
    """A result of `w @ x` is handed out from the pinned pool; feeding it straight
    into `w.T @ ...` (the reference's normal_operator, solvers.py:140-156) takes
    the direct DMA path and gives the same image as a pageable copy."""
    from paper_1310_0956_b200 import build_geometry, build_projector
    n = 512
    w = build_projector(build_geometry(n, 725, 128), precision="float32")
    x = np.random.default_rng(5).random(n * n, dtype=np.float32)
    s = w @ x
    assert torch.from_numpy(s).is_pinned()
    a = w.T @ s
    b = w.T @ s.copy()
    assert np.array_equal(a, b)
