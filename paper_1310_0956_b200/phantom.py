"""Synthetic inputs for the BASELINE configurations (host-side, numpy PCG64).

The reference only ships the fixed Shepp-Logan phantom and uniform white noise
(/root/reference/pkg/src/wmgtomo/phantom.py:17-61); BASELINE.json's configs need
seeded random-ellipse phantoms and Gaussian / Poisson noise, defined here
following the reference's pixel-centre convention (phantom.py:40-49: x = (j +
0.5) 2/n - 1, y = 1 - (i + 0.5) 2/n, row 0 at the top, additive inside
(x_r/a)^2 + (y_r/b)^2 <= 1) and SURVEY.md s8(d):

  ellipse parameters, drawn as arrays in this order from default_rng(seed):
    r = 0.7 sqrt(U), phi = 2 pi U  (centre uniform in the disk r < 0.7),
    a ~ U[0.05, 0.4], b ~ U[0.05, 0.4], rotation ~ U[0, pi),
    value ~ U[lo, hi]  ([-0.3, 1.0] by default; [0, 1] for config 2)
  seeds: config c uses 1000 c + slice for the phantom and + 500 for the noise.

These are input generators (not on the hot path); ``error_metrics`` has a
device twin used inside the solver loops (``solvers._ErrorTracker``).
"""
from __future__ import annotations

import numpy as np

ELLIPSES = (
    (1.0, 0.6900, 0.9200, 0.00, 0.0000, 0.0),
    (-0.8, 0.6624, 0.8740, 0.00, -0.0184, 0.0),
    (-0.2, 0.1100, 0.3100, 0.22, 0.0000, -18.0),
    (-0.2, 0.1600, 0.4100, -0.22, 0.0000, 18.0),
    (0.1, 0.2100, 0.2500, 0.00, 0.3500, 0.0),
    (0.1, 0.0460, 0.0460, 0.00, 0.1000, 0.0),
    (0.1, 0.0460, 0.0460, 0.00, -0.1000, 0.0),
    (0.1, 0.0460, 0.0230, -0.08, -0.6050, 0.0),
    (0.1, 0.0230, 0.0230, 0.00, -0.6060, 0.0),
    (0.1, 0.0230, 0.0460, 0.06, -0.6050, 0.0),
)


def _grid(n):
    xs = (np.arange(n) + 0.5) * (2.0 / n) - 1.0
    ys = 1.0 - (np.arange(n) + 0.5) * (2.0 / n)
    return np.meshgrid(xs, ys)


def _paint(n, ellipses_rad):
    x, y = _grid(n)
    img = np.zeros((n, n))
    for value, a, b, x0, y0, phi in ellipses_rad:
        cp, sp_ = np.cos(phi), np.sin(phi)
        xr = (x - x0) * cp + (y - y0) * sp_
        yr = -(x - x0) * sp_ + (y - y0) * cp
        img[(xr / a) ** 2 + (yr / b) ** 2 <= 1.0] += value
    return img.ravel()


def shepp_logan(n: int) -> np.ndarray:
    """Modified Shepp-Logan at pixel centres (phantom.py:31-50)."""
    if n < 1:
        raise ValueError("n must be >= 1")
    return _paint(n, [(v, a, b, x0, y0, np.deg2rad(d)) for v, a, b, x0, y0, d in ELLIPSES])


def random_ellipses(n: int, count: int, seed: int, value_range=(-0.3, 1.0)) -> np.ndarray:
    """Seeded sum of ``count`` random ellipses (BASELINE configs 0/1/2/4)."""
    if n < 1 or count < 0:
        raise ValueError("n must be >= 1 and count >= 0")
    rng = np.random.default_rng(seed)
    r = 0.7 * np.sqrt(rng.uniform(0.0, 1.0, count))
    phi = 2.0 * np.pi * rng.uniform(0.0, 1.0, count)
    a = rng.uniform(0.05, 0.4, count)
    b = rng.uniform(0.05, 0.4, count)
    rot = rng.uniform(0.0, np.pi, count)
    val = rng.uniform(value_range[0], value_range[1], count)
    ell = [(val[i], a[i], b[i], r[i] * np.cos(phi[i]), r[i] * np.sin(phi[i]), rot[i])
           for i in range(count)]
    return _paint(n, ell)


def seeded_uniform(count: int, seed: int) -> np.ndarray:
    """sparse_kernels.py:78-92: PCG64 uniform on the open interval (-1, 1)."""
    if count < 0:
        raise ValueError("count must be nonnegative")
    rng = np.random.default_rng(seed)
    u = rng.uniform(-1.0, 1.0, size=count)
    while True:
        bad = u <= -1.0
        if not bad.any():
            return u
        u[bad] = rng.uniform(-1.0, 1.0, size=int(bad.sum()))


def add_noise(b, alpha: float, seed: int) -> np.ndarray:
    """b + alpha * U(-1,1) * max|b| (phantom.py:53-61)."""
    if alpha < 0:
        raise ValueError("alpha must be nonnegative")
    b = np.asarray(b, dtype=np.float64)
    if alpha == 0:
        return b.copy()
    return b + alpha * seeded_uniform(b.size, seed) * np.abs(b).max()


def add_gaussian_noise(b, sigma_rel: float, seed: int) -> np.ndarray:
    """b + sigma_rel * max|b| * N(0, 1) (configs 1 and 4)."""
    if sigma_rel < 0:
        raise ValueError("sigma_rel must be nonnegative")
    b = np.asarray(b, dtype=np.float64)
    rng = np.random.default_rng(seed)
    return b + sigma_rel * np.abs(b).max() * rng.standard_normal(b.size)


def poisson_log_data(b, incident: float, mu: float, seed: int) -> np.ndarray:
    """counts ~ Poisson(I0 exp(-mu b)); data = -ln(max(counts, 1) / I0) (config 2).

    mu converts pixel-unit line integrals to attenuation; SURVEY.md s8(d) fixes
    mu = 2/n (the physical pixel size of the [-1,1]^2 phantom).
    """
    b = np.asarray(b, dtype=np.float64)
    rng = np.random.default_rng(seed)
    counts = rng.poisson(incident * np.exp(-mu * b))
    return -np.log(np.maximum(counts, 1) / incident) / mu


def error_metrics(x, x_ex):
    """Relative L2 and L-infinity errors of x against x_ex (phantom.py:64-75)."""
    x = np.asarray(x, dtype=np.float64)
    x_ex = np.asarray(x_ex, dtype=np.float64)
    if x.shape != x_ex.shape:
        raise ValueError("error_metrics: length mismatch")
    norm2 = np.linalg.norm(x_ex)
    norminf = np.abs(x_ex).max() if x_ex.size else 0.0
    if norm2 == 0.0:
        raise ValueError("error_metrics: exact image is identically zero")
    e = x - x_ex
    return float(np.linalg.norm(e) / norm2), float(np.abs(e).max() / norminf)
