"""ORACLE fixture generator (test infrastructure only; run in the build container, where the
read-only reference lives at /root/reference). Writes tests/golden/*.npz.

Every σ fixture is produced by the reference's own code (pseudospec.core, imported from
/root/reference/pkg/src, BLAS pinned to one thread) for real A, and by the restatement
oracle/sigma_oracle.smin_restated (the same numpy zgesdd call without the real cast,
core.py:112-119) for the complex configs C3/C5, which the reference cannot evaluate.
The guided-path fixtures (K2) come from the reference's pipeline.hierarchical_predict /
predicted_region with a bundle trained *by the reference* (network.train, calibrate_threshold)
on a seeded Grcar-family corpus (see train_grcar_bundle).

The writer fixtures (io) are the reference's own io.write_field_csv / write_mask_csv bytes; the
calibration fixture (calib) is the reference's calibrate_threshold on a small validation corpus.

Usage:  python oracle/make_golden.py sigma|model|guided|io|calib|all
"""

from __future__ import annotations

import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import numpy as np
from threadpoolctl import threadpool_limits

ROOT = Path(__file__).resolve().parent.parent
REF = Path("/root/reference/pkg/src")
GOLD = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(REF))

from oracle.sigma_oracle import smin_restated  # noqa: E402
from paper_2605_04550_b200 import configs  # noqa: E402


def _ref_chunk(args):
    A, zs = args
    from pseudospec import core as rcore
    with threadpool_limits(1):
        return rcore.smin_many(A, zs, chunk=1)


def _restated_chunk(args):
    A, zs = args
    return smin_restated(A, zs)


def _pool(fn, A, zs, procs=8):
    chunks = [c for c in np.array_split(zs, max(1, min(procs * 2, zs.size))) if c.size]
    with ProcessPoolExecutor(max_workers=procs) as ex:
        parts = list(ex.map(fn, [(A, c) for c in chunks]))
    return np.concatenate(parts)


def gen_sigma():
    from pseudospec import core as rcore
    GOLD.mkdir(parents=True, exist_ok=True)
    # C1: the reference's full_pseudospectrum on the exact config grid
    cfg = configs.CONFIGS["C1"]
    A = cfg.matrix().todense().real.copy()
    t = time.time()
    with threadpool_limits(1):
        fld = rcore.full_pseudospectrum(A, rcore.make_grid(-1, 3, -3.5, 3.5, 50, 50))
    np.savez_compressed(GOLD / "c1_full.npz", values=fld.values, grid=np.array([-1, 3, -3.5, 3.5, 50, 50.0]),
                        norm2=np.linalg.norm(A, 2))
    print("c1", time.time() - t, flush=True)
    # demo 01: nilpotent shift n=32 on [-1.5,1.5]^2 120x120 (demos/01_sensitivity_basics.py:21-47)
    A01 = np.diag(np.ones(31), k=-1)
    with threadpool_limits(1):
        f01 = rcore.full_pseudospectrum(A01, rcore.make_grid(-1.5, 1.5, -1.5, 1.5, 120, 120))
    shipped = Path("/root/reference/pkg/demos/output_01_field.csv")
    same = None
    if shipped.exists():
        from pseudospec.io import write_field_csv
        tmp = Path("/tmp/_demo01.csv")
        write_field_csv(tmp, f01)
        same = tmp.read_bytes() == shipped.read_bytes()
    np.savez_compressed(GOLD / "demo01_field.npz", values=f01.values,
                        csv_byte_identical=np.array(bool(same)))
    print("demo01 byte-identical to shipped CSV:", same, flush=True)
    # C2 sample (real Grcar n=400): reference smin_many
    for name, count, seed, fn in (("C2", 480, 21, _ref_chunk), ("C3", 192, 31, _restated_chunk),
                                  ("C4", 48, 41, _ref_chunk)):
        cfg = configs.CONFIGS[name]
        Ad = cfg.matrix().todense()
        if np.all(Ad.imag == 0):
            Ad = Ad.real.copy()
        idx, zs = configs.sample_points(cfg, count, seed)
        t = time.time()
        want = _pool(fn, Ad, zs)
        np.savez_compressed(GOLD / f"{name.lower()}_sample.npz", idx=idx, zs=zs, sigma=want,
                            norm2=np.linalg.norm(Ad, 2), kind=np.array("reference" if fn is _ref_chunk else "restated"))
        print(name, count, time.time() - t, flush=True)
    # C5: 4 of the 64 matrices, 6 grid shifts each (restated; n=4000 dense SVDs)
    cfg = configs.CONFIGS["C5"]
    rows = []
    for m in (0, 1, 17, 63):
        Ad = cfg.matrix(m).todense()
        idx, zs = configs.sample_points(cfg, 6, 500 + m)
        t = time.time()
        want = _pool(_restated_chunk, Ad, zs, procs=6)
        rows.append((m, idx, zs, want, np.linalg.norm(Ad, 2)))
        print("C5", m, time.time() - t, flush=True)
    np.savez_compressed(GOLD / "c5_sample.npz", matrices=np.array([r[0] for r in rows]),
                        idx=np.stack([r[1] for r in rows]), zs=np.stack([r[2] for r in rows]),
                        sigma=np.stack([r[3] for r in rows]), norm2=np.array([r[4] for r in rows]))
    gen_small()


def gen_small():
    """Small random banded {-1,0,1} matrices (tests/test_acceptance.py:53-70 style), reference smin_many."""
    from pseudospec import core as rcore
    rng = np.random.default_rng(10)
    mats, zss, sig, ns = [], [], [], []
    for _ in range(30):
        n = int(rng.integers(4, 17))
        beta = int(rng.integers(1, min(4, n - 1) + 1))
        A = rng.integers(-1, 2, size=(n, n)).astype(float)
        i = np.arange(n)
        A[np.abs(i[:, None] - i[None, :]) > beta] = 0.0
        zs = rng.uniform(-4, 4, 40) + 1j * rng.uniform(-4, 4, 40)
        with threadpool_limits(1):
            s = rcore.smin_many(A, zs)
        Ap = np.zeros((16, 16))
        Ap[:n, :n] = A
        mats.append(Ap); zss.append(zs); sig.append(s); ns.append(n)
    np.savez_compressed(GOLD / "small_random.npz", A=np.stack(mats), zs=np.stack(zss), sigma=np.stack(sig),
                        n=np.array(ns))
    print("small random done", flush=True)


# ------------------------------------------------------------------ guided path (K2)
def grcar_family(count, seed, n_choices=(32, 40, 48, 56, 64)):
    """Seeded Grcar-family corpus: Grcar(n, k) with random +-10% perturbations of the band
    coefficients (real), as CorpusMatrix entries of the reference."""
    from pseudospec.generate import CorpusMatrix, mix64
    out = []
    for i in range(count):
        child = mix64(seed, i)
        rng = np.random.default_rng(np.random.PCG64(child))
        n = int(rng.choice(n_choices))
        k = int(rng.integers(2, 5))
        A = -np.diag(np.ones(n - 1), -1) * (1 + 0.1 * rng.uniform(-1, 1))
        for j in range(0, k + 1):
            A += np.diag(np.ones(n - j), j) * (1 + 0.1 * rng.uniform(-1, 1))
        out.append(CorpusMatrix(index=i, seed=child, matrix=A, bandwidth=k, kappa=float(np.linalg.cond(A))))
    return out


def train_grcar_bundle():
    from pseudospec import TrainConfig, build_dataset, calibrate_threshold, make_grid, save_model, train
    grid = make_grid(-1, 3, -3.5, 3.5, 48, 48)
    eps = 0.01
    tr = grcar_family(80, seed=7001)
    va = grcar_family(12, seed=7002)
    t = time.time()
    ds = build_dataset(tr, grid, eps, seed=7003, workers=8)
    print("dataset", len(ds), int(ds.labels.sum()), time.time() - t, flush=True)
    for seed in (42, 43, 44):
        bundle, hist = train(ds, TrainConfig(max_epochs=25, patience=5, seed=seed, batch_size=512))
        rep = calibrate_threshold(bundle, va, grid, eps, workers=8)
        print("seed", seed, "epochs", len(hist), "passed", rep.passed, rep.tau_star, flush=True)
        if rep.passed:
            bundle.tau_star = rep.tau_star
            bundle.meta.update({"train_seed": seed, "corpus": "grcar_family(80, 7001)", "grid": "48x48 C2 box",
                                "eps": eps})
            save_model(bundle, "/tmp/model_grcar.json")
            from pseudospec.network import PARAM_SHAPES
            np.savez_compressed(GOLD / "model_grcar.npz",
                                **{k: getattr(bundle.params, k) for k in PARAM_SHAPES},
                                feature_mean=bundle.feature_mean, feature_std=bundle.feature_std,
                                tau_star=np.array(bundle.tau_star), meta=np.array(json.dumps(bundle.meta)))
            return bundle
    raise SystemExit("calibration failed for every seed")


def load_bundle_npz():
    from pseudospec.network import PARAM_SHAPES, ModelBundle, ModelParams
    z = np.load(GOLD / "model_grcar.npz")
    params = ModelParams(**{k: z[k] for k in PARAM_SHAPES})
    return ModelBundle(params=params, feature_mean=z["feature_mean"], feature_std=z["feature_std"],
                       tau_star=float(z["tau_star"]))


def gen_guided():
    from pseudospec import pipeline, features
    from pseudospec.core import make_grid
    bundle = load_bundle_npz()
    cfg = configs.CONFIGS["C2"]
    A = cfg.matrix().todense().real.copy()
    grid = make_grid(-1, 3, -3.5, 3.5, 200, 200)
    with threadpool_limits(1):
        t = time.time()
        prob, n_evals = pipeline.hierarchical_predict(bundle, A, grid, stride=4, probe_seed=0)
        region = pipeline.predicted_region(prob, bundle.tau_star)
        gf = features.global_features(A, probe_seed=0)
        rng = np.random.default_rng(99)
        zs = grid.points().ravel()[rng.choice(grid.size, 512, replace=False)]
        p_pts = pipeline._predict_points(bundle, gf, zs)
        print("guided", time.time() - t, "evals", n_evals, "region frac", region.mean(), flush=True)
    np.savez_compressed(GOLD / "c2_guided.npz", prob=prob, n_evals=n_evals, region=region,
                        f30=gf.values, eig=gf.eigvals, sample_zs=zs, sample_prob=p_pts, tau=bundle.tau_star)
    # a second, smaller case: C1 (Grcar n=100) so tests stay fast
    A1 = configs.CONFIGS["C1"].matrix().todense().real.copy()
    g1 = make_grid(-1, 3, -3.5, 3.5, 50, 50)
    with threadpool_limits(1):
        prob1, ne1 = pipeline.hierarchical_predict(bundle, A1, g1, stride=4, probe_seed=0)
        reg1 = pipeline.predicted_region(prob1, bundle.tau_star)
        gf1 = features.global_features(A1, probe_seed=0)
        pm1 = pipeline.predict_map(bundle, A1, g1, probe_seed=0)
    np.savez_compressed(GOLD / "c1_guided.npz", prob=prob1, n_evals=ne1, region=reg1, f30=gf1.values,
                        eig=gf1.eigvals, dense=pm1, tau=bundle.tau_star)
    print("c1 guided evals", ne1, "region frac", reg1.mean(), flush=True)


def gen_wide():
    """Larger seeded subsets at SURVEY 8(c)'s sizes: C3 1,024 points (restated; complex A) and
    C4 256 points (the reference's smin_many; real A)."""
    for name, count, seed, fn in (("C3", 1024, 32, _restated_chunk), ("C4", 256, 42, _ref_chunk)):
        cfg = configs.CONFIGS[name]
        Ad = cfg.matrix().todense()
        if np.all(Ad.imag == 0):
            Ad = Ad.real.copy()
        idx, zs = configs.sample_points(cfg, count, seed)
        t = time.time()
        want = _pool(fn, Ad, zs, procs=os.cpu_count() or 8)
        np.savez_compressed(GOLD / f"{name.lower()}_wide.npz", idx=idx, zs=zs, sigma=want,
                            norm2=np.linalg.norm(Ad, 2), kind=np.array("reference" if fn is _ref_chunk else "restated"))
        print(name, "wide", count, time.time() - t, flush=True)


def special_field_values():
    """A 6x7 field covering the writer's special cases (exact 0 -> -inf, NaN, inf, subnormal,
    extremes, values needing all 17 digits)."""
    v = np.array([0.0, np.nan, np.inf, 5e-324, 1e-320, 2.2250738585072014e-308, 1e-300, 1e-5, 1e-4, 0.1, 1.0,
                  1.0000000000000002, 3.141592653589793, 10.0, 100.0, 1e15, 1e16, 1e17, 1.2345678901234567e21,
                  1.7976931348623157e308, 0.30000000000000004, 2.5, 1e22, 9.999999999999999e22, 123456.789,
                  7.0e-5, 6.02214076e23, 1.6e-19, 0.5, 0.25, 0.125, 4.9406564584124654e-324, 1e-7,
                  0.9999999999999999, 12.0, 1e5, 65504.0, 3e-3, 2.0 ** -40, 2.0 ** 60, 7.77e-7, 42.0])
    return v.reshape(6, 7)


def gen_io():
    import hashlib
    import tempfile
    from pseudospec import io as rio
    from pseudospec.core import SigmaField, make_grid
    out = {}
    with tempfile.TemporaryDirectory() as td:
        demo = np.load(GOLD / "demo01_field.npz")["values"]
        g = make_grid(-1.5, 1.5, -1.5, 1.5, 120, 120)
        rio.write_field_csv(f"{td}/demo.csv", SigmaField(g, demo))
        data = open(f"{td}/demo.csv", "rb").read()
        shipped = Path("/root/reference/pkg/demos/output_01_field.csv").read_bytes()
        out["demo01_sha256"] = np.array(hashlib.sha256(data).hexdigest())
        out["demo01_matches_shipped"] = np.array(data == shipped)
        gs = make_grid(-2.0, 7.5, -0.3, 1e-3, 7, 6)
        rio.write_field_csv(f"{td}/special.csv", SigmaField(gs, special_field_values()))
        out["special_csv"] = np.frombuffer(open(f"{td}/special.csv", "rb").read(), dtype=np.uint8)
        rng = np.random.default_rng(5)
        mask = rng.random((9, 11)) < 0.4
        gm = make_grid(-1.0, 3.0, -3.5, 3.5, 11, 9)
        rio.write_mask_csv(f"{td}/mask.csv", mask, gm)
        out["mask"] = mask
        out["mask_csv"] = np.frombuffer(open(f"{td}/mask.csv", "rb").read(), dtype=np.uint8)
    np.savez_compressed(GOLD / "io_writers.npz", **out)
    print("io: demo01 matches shipped", bool(out["demo01_matches_shipped"]), flush=True)


def gen_calib():
    from pseudospec import calibrate_threshold, make_grid
    bundle = load_bundle_npz()
    grid = make_grid(-1, 3, -3.5, 3.5, 48, 48)
    va = grcar_family(4, seed=7002)
    with threadpool_limits(1):
        rep = calibrate_threshold(bundle, va, grid, 0.01, workers=1)
    mats = np.empty(len(va), dtype=object)
    for i, e in enumerate(va):
        mats[i] = e.matrix
    np.savez_compressed(GOLD / "calib_grcar.npz", recalls=rep.recalls, median=rep.median_recall,
                        p10=rep.p10_recall, tau_star=np.array(np.nan if rep.tau_star is None else rep.tau_star),
                        passed=np.array(rep.passed), probe_seeds=np.array([e.probe_seed for e in va]),
                        indices=np.array([e.index for e in va]),
                        **{f"matrix_{i}": e.matrix for i, e in enumerate(va)})
    print("calib: passed", rep.passed, rep.tau_star, flush=True)


def gen_c5_strat(maps_path="gpurun_out/c5_maps.npz", per_matrix=64, procs=6):
    """C5 parity pinned on meaningful points: for each of 4 matrices, 64 grid shifts stratified by what
    they exercise, with sigma from the restated zgesdd oracle (complex A). Strata (per matrix):
      24  bisection-engine points with sigma >= the parity floor 1e-5 ||A||_2 (the general-band kernel)
      16  points straddling the engine split sigma = tau S(z) (tau = 1e-3, S = |z| + sqrt(||A||_1 ||A||_inf)),
          8 on each side
      12  points within 20% of an eps level (1e-1, 1e-2, 1e-3; 4 each)
      12  Lanczos-engine points with sigma >= the floor
    The strata are chosen from a full C5 sigma map computed by this repo's GPU evaluator
    (tools/c5_maps.py); that map only picks *which* shifts to test — every fixture value is the
    oracle's zgesdd (oracle/sigma_oracle.smin_restated)."""
    cfg = configs.CONFIGS["C5"]
    z = np.load(maps_path)
    pts = cfg.grid.points().ravel()
    rows = []
    for m in (int(x) for x in z["matrices"]):
        A = cfg.matrix(m)
        Ad = A.todense()
        n2 = np.linalg.norm(Ad, 2)
        floor = 1e-5 * n2
        anorm = np.sqrt(np.abs(Ad).sum(0).max() * np.abs(Ad).sum(1).max())
        s = z[f"sigma_{m}"].astype(float).ravel()
        st = z[f"status_{m}"].ravel()
        split = 1e-3 * (np.abs(pts) + anorm)
        rng = np.random.default_rng(np.random.PCG64(configs.mix64(5005, m)))
        pick = []

        def take(cand, k):
            cand = np.setdiff1d(cand, np.array(pick, dtype=np.int64))
            sel = rng.choice(cand, size=min(k, cand.size), replace=False) if cand.size else np.zeros(0, int)
            pick.extend(int(c) for c in sel)

        take(np.flatnonzero((st == 1) & (s >= floor)), 24)
        take(np.flatnonzero((s > 0.5 * split) & (s < split)), 8)
        take(np.flatnonzero((s >= split) & (s < 2 * split)), 8)
        for e in (1e-1, 1e-2, 1e-3):
            take(np.flatnonzero(np.abs(s / e - 1) < 0.2), 4)
        take(np.flatnonzero((st == 0) & (s >= floor)), per_matrix - len(pick))
        idx = np.sort(np.array(pick, dtype=np.int64))
        zs = pts[idx]
        t = time.time()
        want = _pool(_restated_chunk, Ad, zs, procs=procs)
        rows.append((m, idx, zs, want, n2))
        print("C5 strat", m, idx.size, "above floor", int((want >= floor).sum()), time.time() - t, flush=True)
        np.savez_compressed(GOLD / "c5_strat.npz", matrices=np.array([r[0] for r in rows]),
                            idx=np.stack([r[1] for r in rows]), zs=np.stack([r[2] for r in rows]),
                            sigma=np.stack([r[3] for r in rows]), norm2=np.array([r[4] for r in rows]),
                            tau=np.array(1e-3))


def _random_bundle(ps, seed, tau):
    rng = np.random.default_rng(seed)
    params = ps.ModelParams(**{k: rng.standard_normal(s) * 0.1 for k, s in ps.network.PARAM_SHAPES.items()})
    return ps.ModelBundle(params=params, feature_mean=np.zeros(33), feature_std=np.ones(33), tau_star=tau)


def gen_pipeline():
    """Reference-made fixtures for the shim-level GPU tests, so they also run where the reference package
    is absent (the GPU box):
      shim_pipeline.npz  the reference's benchmark() / hybrid_pseudospectrum() / full_pseudospectrum() on
                         3 generated n=24 matrices, 40x40 grid, eps 0.05, a seeded random bundle (tau 0.3)
      dataset_labels.npz the reference's build_dataset() (its largest sigma consumer, pipeline.py:128-166)
                         on 4 generated n=32 matrices, 36x36 grid, eps 0.05, seed 5
    The inputs (matrices, probe seeds, bundle parameters) are stored with the outputs."""
    import pseudospec as ps
    from pseudospec import pipeline as rpl
    corpus = ps.generate_corpus(ps.GenSpec(n=24, seed=11), 3)
    grid = ps.make_grid(-4, 4, -4, 4, 40, 40)
    bundle = _random_bundle(ps, 0, 0.3)
    out = {"grid": np.array([-4, 4, -4, 4, 40, 40.0]), "eps": np.array(0.05), "tau_star": np.array(0.3)}
    for k in ps.network.PARAM_SHAPES:
        out[f"p_{k}"] = np.asarray(getattr(bundle.params, k))
    with threadpool_limits(1):
        records, base = rpl.benchmark(bundle, corpus, grid, eps=0.05, baseline=True)
        for i, e in enumerate(corpus):
            out[f"matrix_{i}"] = e.matrix
            out[f"probe_seed_{i}"] = np.array(e.probe_seed)
            out[f"full_{i}"] = ps.core.full_pseudospectrum(e.matrix, grid).values
            res = rpl.hybrid_pseudospectrum(bundle, e.matrix, grid, eps=0.05, probe_seed=e.probe_seed)
            out[f"region_{i}"] = res.region
            out[f"prob_{i}"] = res.prob_field
            out[f"hybrid_{i}"] = res.field.values
            out[f"n_evals_{i}"] = np.array(res.nn_evaluations)
            m = records[i].metrics
            out[f"metrics_{i}"] = np.array([m.accuracy, m.precision, m.recall, m.coverage, m.grid_fraction,
                                            m.tp, m.fp, m.fn], dtype=float)
            out[f"mae_{i}"] = np.array(records[i].mae_log10_smin)
    out["count"] = np.array(len(corpus))
    np.savez_compressed(GOLD / "shim_pipeline.npz", **out)
    print("shim_pipeline: mae", [float(r.mae_log10_smin) for r in records], flush=True)

    corpus = ps.generate_corpus(ps.GenSpec(n=32, seed=21), 4)
    grid = ps.make_grid(-4, 4, -4, 4, 36, 36)
    with threadpool_limits(1):
        ds = rpl.build_dataset(corpus, grid, eps=0.05, seed=5)
    out = {"grid": np.array([-4, 4, -4, 4, 36, 36.0]), "eps": np.array(0.05), "count": np.array(len(corpus)),
           "xy": ds.xy, "features": ds.features, "labels": ds.labels, "matrix_ids": ds.matrix_ids}
    for i, e in enumerate(corpus):
        out[f"matrix_{i}"] = e.matrix
        out[f"index_{i}"] = np.array(e.index)
        out[f"probe_seed_{i}"] = np.array(e.probe_seed)
    np.savez_compressed(GOLD / "dataset_labels.npz", **out)
    print("dataset_labels:", ds.labels.size, "samples,", int(ds.labels.sum()), "positive", flush=True)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if what == "pipeline":
        gen_pipeline()
    if what in ("sigma", "all"):
        gen_sigma()
    if what == "small":
        gen_small()
    if what in ("model", "all"):
        train_grcar_bundle()
    if what in ("guided", "all"):
        gen_guided()
    if what == "wide":
        gen_wide()
    if what in ("io", "all"):
        gen_io()
    if what in ("calib", "all"):
        gen_calib()
    if what == "c5strat":
        gen_c5_strat()
