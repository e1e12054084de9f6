"""ORACLE pinning (CPU): the restatement in oracle/sigma_oracle.py reproduces, bit for bit, the
fixtures that the reference itself produced (oracle/make_golden.py), and the reference's own
golden vector (demos/output_01_field.csv) regenerates byte-identically."""

import numpy as np
import pytest

from oracle.sigma_oracle import floored_rel_err, smin_gesvd, smin_restated
from paper_2605_04550_b200 import configs


def test_demo01_golden_csv_regenerates_byte_identically(gold):
    z = gold("demo01_field.npz")
    assert bool(z["csv_byte_identical"]), "reference did not reproduce demos/output_01_field.csv"
    assert z["values"].shape == (120, 120)
    assert int((z["values"] == 0.0).sum()) == 85  # the 85 '-inf' rows of the shipped CSV


def test_oracle_reproduces_demo01_bitwise(gold):
    want = gold("demo01_field.npz")["values"]
    A = np.diag(np.ones(31), k=-1)
    g = configs.make_grid(-1.5, 1.5, -1.5, 1.5, 120, 120)
    pts = g.points().ravel()
    rng = np.random.default_rng(0)
    idx = np.concatenate([np.flatnonzero(want.ravel() == 0.0)[:10], rng.choice(pts.size, 90, replace=False)])
    got = smin_restated(A, pts[idx])
    assert np.array_equal(got, want.ravel()[idx])


def test_oracle_reproduces_c1_bitwise(gold):
    z = gold("c1_full.npz")
    A = configs.CONFIGS["C1"].matrix().todense().real
    pts = configs.CONFIGS["C1"].grid.points().ravel()
    idx = np.arange(0, pts.size, 7)
    assert np.array_equal(smin_restated(A, pts[idx]), z["values"].ravel()[idx])


def test_oracle_reproduces_c2_sample_bitwise(gold):
    z = gold("c2_sample.npz")
    A = configs.CONFIGS["C2"].matrix().todense().real
    assert np.array_equal(configs.CONFIGS["C2"].grid.points().ravel()[z["idx"]], z["zs"])
    got = smin_restated(A, z["zs"][:24])
    assert np.array_equal(got, z["sigma"][:24])


def test_oracle_reproduces_small_random_bitwise(gold):
    z = gold("small_random.npz")
    for t in range(0, len(z["A"]), 3):
        n = int(z["n"][t])
        A = z["A"][t][:n, :n]
        assert np.array_equal(smin_restated(A, z["zs"][t]), z["sigma"][t])


def test_oracle_c3_restatement_matches_fixture(gold):
    z = gold("c3_sample.npz")
    A = configs.CONFIGS["C3"].matrix().todense()
    got = smin_restated(A, z["zs"][:3])
    assert np.array_equal(got, z["sigma"][:3])


def test_oracle_independent_gesvd_route(gold):
    """tests/test_core.py:82-103 of the reference: the gesvd driver agrees at 1e-10*max(1, want)."""
    z = gold("small_random.npz")
    worst = 0.0
    for t in range(0, len(z["A"]), 5):
        n = int(z["n"][t])
        A = z["A"][t][:n, :n]
        got = smin_gesvd(A, z["zs"][t][:10])
        want = z["sigma"][t][:10]
        worst = max(worst, float(np.max(np.abs(got - want) / np.maximum(1.0, want))))
    assert worst < 1e-10


def test_fixture_grids_match_configs(gold):
    for name in ("c2", "c3", "c4"):
        z = gold(f"{name}_sample.npz")
        cfg = configs.CONFIGS[name.upper()]
        assert np.array_equal(cfg.grid.points().ravel()[z["idx"]], z["zs"])
    z = gold("c5_sample.npz")
    pts = configs.CONFIGS["C5"].grid.points().ravel()
    for r in range(len(z["matrices"])):
        assert np.array_equal(pts[z["idx"][r]], z["zs"][r])


def test_parity_metric_is_floored():
    got = np.array([1e-20, 1.0 + 1e-12, 0.5])
    want = np.array([0.0, 1.0, 0.5])
    e = floored_rel_err(got, want, 1e-5)
    assert e[0] <= 1e-9 and e[1] == pytest.approx(1e-12, rel=1e-3) and e[2] == 0.0


def test_restatement_equals_live_reference(reference_pkg):
    """Cross-check against the reference package itself (present in the build container)."""
    from pseudospec import core as rcore
    rng = np.random.default_rng(3)
    for _ in range(4):
        n = int(rng.integers(5, 20))
        A = rng.integers(-1, 2, size=(n, n)).astype(float)
        i = np.arange(n)
        A[np.abs(i[:, None] - i[None, :]) > 2] = 0.0
        zs = rng.uniform(-3, 3, 12) + 1j * rng.uniform(-3, 3, 12)
        from threadpoolctl import threadpool_limits
        with threadpool_limits(1):
            want = rcore.smin_many(A, zs)
        assert np.array_equal(smin_restated(A, zs), want)


def test_mix64_matches_reference(reference_pkg):
    from pseudospec.generate import mix64 as rmix
    for s, i in ((0, 0), (7, 3), (2**63, 17), (260504550, 5)):
        assert configs.mix64(s, i) == rmix(s, i)
