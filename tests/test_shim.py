"""shim.install(): the reference package's own entry points rerouted onto the B200 evaluator."""

import numpy as np
import pytest


def test_install_rebinds_and_uninstall_restores(refpkg_any):
    import importlib

    from paper_2605_04550_b200 import shim
    ps = refpkg_any
    importlib.import_module(ps.__name__ + ".cli")
    orig = (ps.core.smin_many, ps.pipeline.full_pseudospectrum, ps.pipeline.restricted_field,
            ps.pipeline._predict_points, ps.cli.full_pseudospectrum)
    shim.install(ps)
    try:
        assert ps.core.smin_many is not orig[0]
        assert ps.pipeline.full_pseudospectrum is ps.core.full_pseudospectrum is ps.cli.full_pseudospectrum
        assert ps.pipeline._predict_points is not orig[3]
    finally:
        shim.uninstall()
    assert (ps.core.smin_many, ps.pipeline.full_pseudospectrum, ps.pipeline.restricted_field,
            ps.pipeline._predict_points, ps.cli.full_pseudospectrum) == orig


def test_shim_keeps_reference_validation(refpkg_any):
    from paper_2605_04550_b200 import shim
    ps = refpkg_any
    shim.install(ps)
    try:
        with pytest.raises(ps.core.ParameterError):
            ps.core.smin_many(np.ones((3, 4)), [1j])
        g = ps.core.make_grid(0, 1, 0, 1, 3, 3)
        with pytest.raises(ps.core.ParameterError):
            ps.core.restricted_field(np.eye(2), g, np.ones((3, 3), dtype=int))
    finally:
        shim.uninstall()


@pytest.mark.gpu
def test_reference_pipeline_runs_on_gpu(gpu, refpkg_any):
    """The reference's own hybrid_pseudospectrum / evaluate / benchmark over the shim: σ equal to the
    reference's zgesdd within the parity gate, restriction exactness bitwise, MAE tripwire 0."""
    from threadpoolctl import threadpool_limits

    from paper_2605_04550_b200 import shim
    ps = refpkg_any
    corpus = ps.generate_corpus(ps.GenSpec(n=24, seed=11), 3)
    grid = ps.make_grid(-4, 4, -4, 4, 40, 40)
    with threadpool_limits(1):
        want = [ps.core.full_pseudospectrum(e.matrix, grid).values for e in corpus]  # original zgesdd path
    rng = np.random.default_rng(0)
    params = ps.ModelParams(**{k: rng.standard_normal(s) * 0.1 for k, s in ps.network.PARAM_SHAPES.items()})
    bundle = ps.ModelBundle(params=params, feature_mean=np.zeros(33), feature_std=np.ones(33), tau_star=0.3)
    shim.install(ps)
    try:
        for e, w in zip(corpus, want):
            got = ps.core.full_pseudospectrum(e.matrix, grid)
            assert isinstance(got, ps.core.SigmaField)
            floor = 1e-5 * np.linalg.norm(e.matrix, 2)
            assert np.max(np.abs(got.values - w) / np.maximum(w, floor)) <= 1e-9
        records, base = ps.pipeline.benchmark(bundle, corpus, grid, eps=0.05, baseline=True)
        assert all(r.mae_log10_smin == 0.0 for r in records)  # pipeline.py:379-385 tripwire
        res = ps.pipeline.hybrid_pseudospectrum(bundle, corpus[0].matrix, grid, eps=0.05,
                                                probe_seed=corpus[0].probe_seed)
        full = ps.core.full_pseudospectrum(corpus[0].matrix, grid)
        assert np.array_equal(res.field.values[res.region], full.values[res.region])
    finally:
        shim.uninstall()


@pytest.mark.gpu
def test_reference_calibrate_and_writers_run_on_gpu(gpu, refpkg_any, tmp_path):
    """The reference's calibrate_threshold (recall loop on the K2 kernel) and CSV writers (native)
    through the shim give the reference's own report and bytes."""
    from threadpoolctl import threadpool_limits

    import importlib

    from paper_2605_04550_b200 import shim
    ps = refpkg_any
    importlib.import_module(ps.__name__ + ".io")
    corpus = ps.generate_corpus(ps.GenSpec(n=24, seed=12), 2)
    grid = ps.make_grid(-4, 4, -4, 4, 30, 30)
    rng = np.random.default_rng(1)
    params = ps.ModelParams(**{k: rng.standard_normal(s) * 0.1 for k, s in ps.network.PARAM_SHAPES.items()})
    bundle = ps.ModelBundle(params=params, feature_mean=np.zeros(33), feature_std=np.ones(33), tau_star=0.3)
    with threadpool_limits(1):
        want = ps.pipeline.calibrate_threshold(bundle, corpus, grid, eps=0.05)
        fld = ps.core.full_pseudospectrum(corpus[0].matrix, grid)
        ps.io.write_field_csv(tmp_path / "ref.csv", fld)
        ps.io.write_mask_csv(tmp_path / "refm.csv", fld.values <= 0.05, grid)
    shim.install(ps)
    try:
        got = ps.pipeline.calibrate_threshold(bundle, corpus, grid, eps=0.05)
        assert isinstance(got, ps.pipeline.CalibrationReport)
        assert np.array_equal(got.recalls, want.recalls) and got.tau_star == want.tau_star
        ps.io.write_field_csv(tmp_path / "ours.csv", fld)
        ps.io.write_mask_csv(tmp_path / "oursm.csv", fld.values <= 0.05, grid)
        assert (tmp_path / "ours.csv").read_bytes() == (tmp_path / "ref.csv").read_bytes()
        assert (tmp_path / "oursm.csv").read_bytes() == (tmp_path / "refm.csv").read_bytes()
    finally:
        shim.uninstall()


@pytest.mark.gpu
def test_reference_build_dataset_labels_on_gpu(gpu, refpkg_any):
    """the reference's build_dataset (its largest σ consumer) through the shim
    gives the same balanced samples, features and labels as its own zgesdd path."""
    from threadpoolctl import threadpool_limits

    from paper_2605_04550_b200 import shim
    ps = refpkg_any
    corpus = ps.generate_corpus(ps.GenSpec(n=32, seed=21), 4)
    grid = ps.make_grid(-4, 4, -4, 4, 36, 36)
    with threadpool_limits(1):
        want = ps.pipeline.build_dataset(corpus, grid, eps=0.05, seed=5)
    shim.install(ps)
    try:
        got = ps.pipeline.build_dataset(corpus, grid, eps=0.05, seed=5)
    finally:
        shim.uninstall()
    for name in ("xy", "features", "labels", "matrix_ids"):
        assert np.array_equal(getattr(got, name), getattr(want, name)), name
