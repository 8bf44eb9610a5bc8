import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN_DIR, "golden.json")) as fh:
        meta = json.load(fh)
    arrays = dict(np.load(os.path.join(GOLDEN_DIR, "golden.npz")))
    return meta, arrays


@pytest.fixture(scope="session")
def oracle_proj():
    from oracle import cproj
    cproj.lib()
    return cproj


def case_geometry(spec):
    """(n, d, angles) of a golden projector case."""
    n, d, m = spec["n"], spec["d"], spec["m"]
    angles = np.arange(m) * (np.pi / m)
    if spec["subset"] is not None:
        angles = angles[np.asarray(spec["subset"])]
    return n, d, angles


def case_vectors(spec, n_rows):
    rs = np.random.default_rng(spec["seed"])
    x = rs.standard_normal(spec["n"] ** 2)
    y = rs.standard_normal(n_rows)
    return x, y


@pytest.fixture(scope="session")
def gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1310_0956_b200 import _native
    _native.load(require_gpu=True)
    return torch
