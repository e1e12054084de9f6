"""Guided-path host logic (CPU): global features, bundle formats, fine-point enumeration."""

import json

import numpy as np
import pytest

from paper_2605_04550_b200 import configs, pipeline
from paper_2605_04550_b200.core import ModelFormatError, ParameterError
from pathlib import Path

GOLD = Path(__file__).resolve().parent / "golden"


def test_global_features_match_fixture_bitwise(gold):
    for name, cfg in (("c1_guided.npz", "C1"), ("c2_guided.npz", "C2")):
        z = gold(name)
        A = configs.CONFIGS[cfg].matrix().todense().real
        gf = pipeline.global_features(A, probe_seed=0)
        assert np.array_equal(gf.values, z["f30"])
        assert np.array_equal(gf.eigvals, z["eig"])


def test_global_features_equal_reference(reference_pkg):
    from pseudospec import features
    rng = np.random.default_rng(4)
    A = rng.integers(-1, 2, size=(24, 24)).astype(float)
    i = np.arange(24)
    A[np.abs(i[:, None] - i[None, :]) > 3] = 0
    a = features.global_features(A, probe_seed=77)
    b = pipeline.global_features(A, probe_seed=77)
    assert np.array_equal(a.values, b.values) and np.array_equal(a.eigvals, b.eigvals)


def test_bundle_packing_order():
    rng = np.random.default_rng(0)
    params = {k: rng.standard_normal(s) for k, s in pipeline.PARAM_SHAPES.items()}
    b = pipeline.ModelBundle(params, np.zeros(33), np.ones(33), 0.1)
    flat = b.packed()
    assert flat.size == pipeline.N_PARAMS == 59841
    off = 0
    for k, s in pipeline.PARAM_SHAPES.items():
        n = int(np.prod(s)) if s else 1
        assert np.array_equal(flat[off:off + n], np.ravel(params[k]))
        off += n


def test_bundle_validation():
    params = {k: np.zeros(s) for k, s in pipeline.PARAM_SHAPES.items()}
    with pytest.raises(ParameterError):
        pipeline.ModelBundle(params, np.zeros(33), np.zeros(33))
    bad = dict(params, w_c1=np.zeros((3, 3)))
    with pytest.raises(ParameterError):
        pipeline.ModelBundle(bad, np.zeros(33), np.ones(33))


def test_load_reference_json_roundtrip(tmp_path, reference_pkg):
    from pseudospec import network
    rb = network.ModelBundle(params=network.init_params(3), feature_mean=np.arange(33.0),
                             feature_std=np.ones(33), tau_star=0.12, meta={"k": 1})
    path = tmp_path / "m.json"
    network.save_model(rb, path)
    ours = pipeline.load_model(path)
    assert ours.tau_star == 0.12 and ours.meta == {"k": 1}
    for k in pipeline.PARAM_SHAPES:
        assert np.array_equal(ours.params[k], getattr(rb.params, k))


def test_load_model_errors(tmp_path):
    p = tmp_path / "x.json"
    p.write_text("{nope")
    with pytest.raises(ModelFormatError):
        pipeline.load_model(p)
    p.write_text(json.dumps({"meta": {"format": "other"}, "feature_norm": {}, "params": {}, "calibration": {}}))
    with pytest.raises(ModelFormatError):
        pipeline.load_model(p)


def test_fixture_bundle_loads():
    b = pipeline.load_npz(GOLD / "model_grcar.npz")
    assert b.tau_star == pytest.approx(0.05)


def test_fine_points_match_reference_enumeration():
    """Same points, same order as pipeline.py:206-215 (incl. partial cells at the border)."""
    rng = np.random.default_rng(2)
    ny, nx, s = 21, 18, 4
    ay, ax = np.arange(0, ny, s), np.arange(0, nx, s)
    flagged = rng.uniform(size=(ay.size, ax.size)) < 0.4
    rows, cols = pipeline._fine_points(flagged, ay, ax, s, ny, nx)
    want = []
    for iy, ix in zip(*np.nonzero(flagged)):
        for r in range(ay[iy], min(ay[iy] + s, ny)):
            for c in range(ax[ix], min(ax[ix] + s, nx)):
                if (r, c) != (ay[iy], ax[ix]):
                    want.append((r, c))
    assert list(zip(rows.tolist(), cols.tolist())) == want


def test_fine_points_vectorised_order():
    """The vectorised fine-point list equals the per-cell loop (pipeline.py:206-215 order), clipped cells too."""
    import numpy as np

    from paper_2605_04550_b200 import pipeline
    rng = np.random.default_rng(3)
    for ny, nx, s in ((50, 50, 4), (37, 53, 4), (512, 512, 4), (9, 7, 3), (5, 5, 4)):
        ay, ax = np.arange(0, ny, s), np.arange(0, nx, s)
        for frac in (0.0, 0.2, 1.0):
            flagged = rng.random((ay.size, ax.size)) < frac
            a = pipeline._fine_points(flagged, ay, ax, s, ny, nx)
            b = pipeline._fine_points_loop(flagged, ay, ax, s, ny, nx)
            assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
