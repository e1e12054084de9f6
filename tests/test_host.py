"""Host-side logic (CPU): grid/field types, masks, dilation, bands, configs, validation."""

import numpy as np
import pytest

from paper_2605_04550_b200 import configs, core
from paper_2605_04550_b200.core import ParameterError


def dilate_bruteforce(mask, k):  # tests/test_core.py:197-205 of the reference, restated
    h = k // 2
    ny, nx = mask.shape
    out = np.zeros_like(mask)
    for i in range(ny):
        for j in range(nx):
            out[i, j] = mask[max(0, i - h):i + h + 1, max(0, j - h):j + h + 1].any()
    return out


class TestGrid:
    def test_default_domain(self):
        g = core.make_grid(-4, 4, -4, 4, 100, 100)
        assert g.size == 10_000
        assert g.xs()[1] - g.xs()[0] == pytest.approx(8 / 99, rel=1e-15)

    def test_points_layout(self):
        g = core.make_grid(0, 1, 0, 1, 2, 2)
        assert set(g.points().ravel().tolist()) == {0, 1j, 1, 1 + 1j}
        g = core.make_grid(-1, 1, -2, 2, 5, 3)
        assert g.points()[2, 4] == 1 + 2j  # rows = imaginary axis

    @pytest.mark.parametrize("bad", [(1, 0, 0, 1, 3, 3), (0, 1, 1, 0, 3, 3), (0, 1, 0, 1, 1, 3), (0, 1, 0, 1, 3, 1)])
    def test_rejects_bad_parameters(self, bad):
        with pytest.raises(ParameterError):
            core.make_grid(*bad)

    def test_endpoints_inclusive(self):
        g = core.make_grid(-2, 3, 0.5, 1.5, 7, 4)
        assert g.xs()[0] == -2 and g.xs()[-1] == 3 and g.ys()[-1] == 1.5


class TestField:
    def test_mask_nan_false_and_eps_positive(self):
        g = core.make_grid(0, 2, -1, 1, 5, 5)
        vals = np.full((5, 5), np.nan)
        vals[1, 1] = 0.0
        f = core.SigmaField(g, vals)
        assert core.sensitive_zone(f, 0.5).sum() == 1
        with pytest.raises(ParameterError):
            core.sensitive_zone(f, 0.0)

    def test_shape_mismatch(self):
        with pytest.raises(ParameterError):
            core.SigmaField(core.make_grid(0, 1, 0, 1, 3, 3), np.ones((2, 3)))


class TestDilate:
    @pytest.mark.parametrize("k", [1, 3, 5, 7])
    @pytest.mark.parametrize("seed", range(4))
    def test_matches_bruteforce(self, k, seed):
        mask = np.random.default_rng(seed).uniform(size=(12, 17)) < 0.1
        assert np.array_equal(core.dilate(mask, k), dilate_bruteforce(mask, k))

    def test_corner_clipping_and_empty(self):
        m = np.zeros((5, 5), bool)
        m[0, 0] = True
        assert core.dilate(m, 5).sum() == 9
        assert core.dilate(np.zeros((4, 6), bool), 5).sum() == 0

    def test_rejects_even(self):
        with pytest.raises(ParameterError):
            core.dilate(np.zeros((3, 3), bool), 4)

    def test_matches_scipy(self):
        from scipy.ndimage import binary_dilation
        m = np.random.default_rng(9).uniform(size=(40, 33)) < 0.05
        assert np.array_equal(core.dilate(m, 5), binary_dilation(m, structure=np.ones((5, 5), bool)))


class TestBands:
    def test_band_roundtrip(self):
        rng = np.random.default_rng(1)
        A = rng.standard_normal((9, 9)) + 1j * rng.standard_normal((9, 9))
        i = np.arange(9)
        A[(i[:, None] - i[None, :] > 2) | (i[None, :] - i[:, None] > 3)] = 0
        assert core.bandwidths(A) == (2, 3)
        bm = core.BandMatrix(core.band_of(A), 2, 3)
        assert np.array_equal(bm.todense(), A)

    def test_grcar_band(self):
        A = configs.grcar_band(6).todense().real
        want = -np.diag(np.ones(5), -1) + sum(np.diag(np.ones(6 - j), j) for j in range(4))
        assert np.array_equal(A, want)

    def test_convdiff(self):
        A = configs.convdiff_band(5).todense().real
        h = 1 / 6
        assert A[1, 0] == pytest.approx(1 / h**2 - 25 / h) and A[0, 1] == pytest.approx(1 / h**2 + 25 / h)

    def test_config_shapes(self):
        for name, (n, kl, ku) in {"C1": (100, 1, 3), "C2": (400, 1, 3), "C3": (1000, 2, 3), "C4": (2000, 1, 1),
                                  "C5": (4000, 3, 3)}.items():
            m = configs.CONFIGS[name].matrix(0)
            assert (m.n, m.kl, m.ku) == (n, kl, ku)
        assert configs.CONFIGS["C5"].grid.size == 1024 * 1024 and configs.CONFIGS["C5"].batch == 64

    def test_c5_matrices_differ_and_are_seeded(self):
        a, b = configs.c5_band(0, 50), configs.c5_band(1, 50)
        assert not np.array_equal(a.band, b.band)
        assert np.array_equal(a.band, configs.c5_band(0, 50).band)


class TestValidation:
    """Argument errors surface as ParameterError before any device work (core.py:112-119)."""

    def test_non_square(self):
        with pytest.raises(ParameterError):
            core.smin_many(np.ones((3, 4)), [1j])

    def test_non_finite(self):
        A = np.eye(3)
        A[0, 0] = np.nan
        with pytest.raises(ParameterError):
            core.smin_many(A, [1j])

    def test_non_finite_shift_is_numerical_error(self):
        """The reference's svd raises LinAlgError on a NaN shift, reported as NumericalError with
        the point index and z (core.py:157-166)."""
        from paper_2605_04550_b200.core import NumericalError
        with pytest.raises(NumericalError, match="point index 1"):
            core.smin_many(np.eye(3), [0.5, np.nan, 1j])
        with pytest.raises(NumericalError):
            core.smin_at(np.eye(3), complex(np.inf, 0))

    def test_too_small(self):
        with pytest.raises(ParameterError):
            core.smin_many(np.eye(1), [0.5])

    def test_bandwidth_limit(self):
        with pytest.raises(ParameterError):
            core.smin_many(np.ones((20, 20)), [1j])

    def test_region_mask_checked(self):
        g = core.make_grid(0, 1, 0, 1, 3, 3)
        with pytest.raises(ParameterError):
            core.restricted_field(np.eye(2), g, np.ones((3, 3), dtype=int))
