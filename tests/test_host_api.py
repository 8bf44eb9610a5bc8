"""Host-side API semantics (no GPU): the reference's own unit tests for the
parts of the API that do not launch kernels (tests/test_geometry.py:31-62,
tests/test_solvers.py:10-40, tests/test_multilevel.py:16-63,
tests/test_phantom.py, tests/test_sparse_kernels.py:75-93), run against the
B200 package."""
import numpy as np
import pytest

from paper_1310_0956_b200 import (BAND_IDS, ConvergenceRecord, Geometry, SolverConfig,
                                  add_gaussian_noise, add_noise, build_geometry,
                                  build_intergrid_set, error_metrics, find_kopt, haar_scaling_1d,
                                  haar_wavelet_1d, poisson_log_data, random_ellipses,
                                  seeded_uniform, shepp_logan)
from paper_1310_0956_b200.geometry import snapped_trig


class TestGeometry:
    def test_angle_grid(self):
        g = build_geometry(8, 8, 4)
        np.testing.assert_allclose(g.angles, [0.0, np.pi / 4, np.pi / 2, 3 * np.pi / 4],
                                   atol=1e-15)
        assert g.n_image == 64 and g.n_data == 32

    def test_rejects_bad_sizes(self):
        for bad in [(0, 8, 4), (8, 0, 4), (8, 8, 0)]:
            with pytest.raises(ValueError):
                build_geometry(*bad)

    def test_rejects_bad_angles(self):
        with pytest.raises(ValueError):
            Geometry(4, 4, 2, angles=np.array([0.0, np.pi]))
        with pytest.raises(ValueError):
            Geometry(4, 4, 2, angles=np.array([0.5, 0.5]))
        with pytest.raises(ValueError):
            Geometry(4, 4, 2, angles=np.array([0.5, 0.2]))

    def test_subset(self):
        g = build_geometry(16, 24, 24)
        s = g.subset([0, 5, 7])
        assert s.n_angles == 3 and np.array_equal(s.angles, g.angles[[0, 5, 7]])

    def test_snapped_trig_matches_oracle(self):
        from oracle import cproj
        for m in (1, 2, 4, 90, 180, 720, 4096):
            a = np.arange(m) * (np.pi / m)
            c1, s1 = snapped_trig(a)
            c2, s2 = cproj.snapped_trig(a)
            assert np.array_equal(c1, c2) and np.array_equal(s1, s2)
        c, s = snapped_trig(np.array([0.0, np.pi / 2]))
        assert (c[0], s[0], c[1], s[1]) == (1.0, 0.0, 0.0, 1.0)


class TestConfigAndRecord:
    def test_config_validation(self):
        with pytest.raises(ValueError):
            SolverConfig(max_iterations=0)
        with pytest.raises(ValueError):
            SolverConfig(residual_tolerance=-1.0)
        with pytest.raises(ValueError):
            SolverConfig(regularization_lambda=-1.0)

    def test_find_kopt_first_minimum(self):
        rec = ConvergenceRecord()
        for k, e in enumerate([1.0, 0.5, 0.2, 0.2, 0.4]):
            rec.log(k, 1.0, e, e, 0.0)
        assert find_kopt(rec) == 2

    def test_find_kopt_requires_errors(self):
        rec = ConvergenceRecord()
        rec.log(0, 1.0, None, None, 0.0)
        with pytest.raises(ValueError):
            find_kopt(rec)


class TestHaar:
    def test_stencils(self):
        s = haar_scaling_1d(4).toarray()
        j = haar_wavelet_1d(4).toarray()
        c = 1.0 / np.sqrt(2.0)
        np.testing.assert_allclose(s, [[c, c, 0, 0], [0, 0, c, c]])
        np.testing.assert_allclose(j, [[c, -c, 0, 0], [0, 0, c, -c]])

    def test_rejects_odd(self):
        for bad in (1, 3, 0):
            with pytest.raises(ValueError):
                haar_scaling_1d(bad)

    @pytest.mark.parametrize("n", [2, 4, 8, 16, 32, 64])
    def test_orthogonality_and_reconstruction(self, n):
        grids = build_intergrid_set(n)
        eye = np.eye(n * n // 4)
        for a in BAND_IDS:
            assert np.abs((grids[a] @ grids[a].T).toarray() - eye).max() <= 1e-14
        for i, a in enumerate(BAND_IDS):
            for b in BAND_IDS[i + 1:]:
                assert np.abs((grids[a] @ grids[b].T).toarray()).max() <= 1e-14
        total = sum((grids[b].T @ grids[b]).toarray() for b in BAND_IDS)
        assert np.abs(total - np.eye(n * n)).max() <= 1e-14

    def test_band_orientation_and_coefficient(self):
        grids = build_intergrid_set(8)
        const_y = np.tile(np.arange(8.0), 8)
        const_x = np.repeat(np.arange(8.0), 8)
        assert np.abs(grids["LH"] @ const_y).max() <= 1e-13
        assert np.abs(grids["LH"] @ const_x).max() > 0.1
        assert np.abs(grids["HL"] @ const_x).max() <= 1e-13
        # the kernels hard-code fl(fl(1/sqrt 2)^2) = 0.4999999999999999
        assert set(np.abs(grids["HH"].data)) == {0.4999999999999999}


class TestPhantomsAndNoise:
    def test_shepp_logan_values(self):
        ph = shepp_logan(64).reshape(64, 64)
        assert ph.min() >= -1e-12 and ph.max() <= 1.0 + 1e-12
        assert ph[0, 0] == 0.0 and ph[32, 32] > 0.0

    def test_random_ellipses_seeded(self):
        a = random_ellipses(64, 10, seed=0)
        assert np.array_equal(a, random_ellipses(64, 10, seed=0))
        assert not np.array_equal(a, random_ellipses(64, 10, seed=1))
        x = np.linspace(-1, 1, 64)
        r = np.hypot(*np.meshgrid((np.arange(64) + 0.5) / 32 - 1, 1 - (np.arange(64) + 0.5) / 32))
        assert np.all(a.reshape(64, 64)[r > 0.7 + 0.4 + 1e-9] == 0.0)   # centres in r < 0.7
        assert x.size == 64

    def test_noise_models(self):
        b = np.linspace(0.0, 10.0, 1000)
        nb = add_noise(b, 0.01, seed=11)
        assert np.abs(nb - b).max() <= 0.01 * 10.0
        assert np.array_equal(nb, add_noise(b, 0.01, seed=11))
        assert np.array_equal(add_noise(b, 0.0, seed=1), b)
        gb = add_gaussian_noise(b, 0.01, seed=1500)
        assert 0.05 < np.std(gb - b) < 0.15
        pb = poisson_log_data(b, 1e5, 2.0 / 64, seed=2500)
        assert np.abs(pb - b).max() < 0.5 * 64

    def test_seeded_uniform_frozen(self):
        np.testing.assert_allclose(seeded_uniform(4, 42),
                                   [0.5479121, -0.12224312, 0.71719584, 0.39473606], atol=1e-8)
        u = seeded_uniform(10000, 0)
        assert u.min() > -1.0 and u.max() < 1.0
        with pytest.raises(ValueError):
            seeded_uniform(-1, 1)

    def test_error_metrics(self):
        x_ex = np.array([1.0, 2.0, 2.0])
        e2, einf = error_metrics(x_ex + np.array([0.0, 0.0, 0.3]), x_ex)
        assert abs(e2 - 0.1) < 1e-15 and abs(einf - 0.15) < 1e-15
        with pytest.raises(ValueError):
            error_metrics(np.zeros(2), np.zeros(2))
        with pytest.raises(ValueError):
            error_metrics(np.zeros(2), np.ones(3))


def test_product_has_no_cpu_fallback():
    """Without a GPU the product path raises instead of computing on the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1310_0956_b200 import build_projector
    with pytest.raises(RuntimeError):
        build_projector(build_geometry(8, 8, 4))
