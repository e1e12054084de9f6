"""Drop-in for the guided (hybrid) path of `pseudospec.pipeline` on K2 + K1.

Mirrors, with the same names, arguments and results:
  _predict_points        pipeline.py:169-172  -> K2 kernel (features g1..g3, standardize,
                                                 Fourier encoding, dual-path SiLU MLP, sigmoid)
  predict_map            pipeline.py:175-179
  hierarchical_predict   pipeline.py:182-224  (coarse anchors, 80th-percentile refinement on
                                                 the host with numpy, fine points on K2)
  predicted_region       pipeline.py:227-231  -> K2 region kernel (>= tau, 5x5 dilation)
  hybrid_pseudospectrum  pipeline.py:273-297  -> K2 + restricted σ sweep on K1
  calibrate_threshold    pipeline.py:241-270  -> full σ maps on K1, dense K2 maps, and the
                                                 90-threshold recall loop in one K2 kernel
and the host inputs they need: global_features (features.py:63-117, O(n^3) per matrix, host
LAPACK as in the reference — SURVEY.md §8(f) row 1) and the model bundle format
(network.py:35-52 PARAM_SHAPES, network.py:430-479 JSON document).
"""

from __future__ import annotations

import ctypes as C
import hashlib
import json
import os
import threading
import time
from collections import OrderedDict
from concurrent.futures import Future, ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

from . import _lib, core
from .configs import mix64
from .core import ComplexGrid, ModelFormatError, ParameterError, SigmaField

TRUTH_DILATION = 3
PRED_DILATION = 5
CAL_TAUS = np.round(np.arange(0.05, 0.95, 0.01), 2)  # pipeline.py:25
COORD_DIM, FEATURE_DIM = 26, 33
PARAM_SHAPES = {
    "w_c1": (64, COORD_DIM), "b_c1": (64,), "w_c2": (64, 64), "b_c2": (64,),
    "w_m1": (128, FEATURE_DIM), "b_m1": (128,), "w_m2": (64, 128), "b_m2": (64,),
    "w_t1": (128, 128), "b_t1": (128,), "w_t2": (128, 128), "b_t2": (128,),
    "w_proj": (64, 128), "b_proj": (64,), "w_head": (64,), "b_head": (),
}
N_PARAMS = 59841


# ----------------------------------------------------------------------------- bundle
@dataclass
class ModelBundle:
    """Trained parameters, feature normalization, calibrated threshold (network.py:308-330)."""

    params: dict
    feature_mean: np.ndarray
    feature_std: np.ndarray
    tau_star: float | None = None
    meta: dict = field(default_factory=dict)

    def __post_init__(self):
        if not isinstance(self.params, dict):  # a reference ModelParams object
            self.params = {k: np.asarray(getattr(self.params, k), dtype=float) for k in PARAM_SHAPES}
        for k, shp in PARAM_SHAPES.items():
            a = np.asarray(self.params[k], dtype=float)
            if a.shape != shp:
                raise ParameterError(f"{k} must have shape {shp}, got {a.shape}")
            self.params[k] = a
        # contiguous copies: the C ABI reads them as raw 33-double arrays
        self.feature_mean = np.ascontiguousarray(self.feature_mean, dtype=float)
        self.feature_std = np.ascontiguousarray(self.feature_std, dtype=float)
        if self.feature_mean.shape != (FEATURE_DIM,) or self.feature_std.shape != (FEATURE_DIM,):
            raise ParameterError("feature statistics must be 33-vectors")
        if np.any(self.feature_std <= 0):
            raise ParameterError("feature_std entries must be positive")

    def packed(self) -> np.ndarray:
        """The 16 arrays concatenated in PARAM_SHAPES order (the C ABI layout)."""
        out = np.concatenate([np.asarray(self.params[k], dtype=float).ravel() for k in PARAM_SHAPES])
        assert out.size == N_PARAMS
        return np.ascontiguousarray(out)

    @classmethod
    def from_reference(cls, bundle) -> "ModelBundle":
        return cls(params=bundle.params, feature_mean=bundle.feature_mean, feature_std=bundle.feature_std,
                   tau_star=bundle.tau_star, meta=dict(bundle.meta))


def load_model(path) -> ModelBundle:
    """Read the reference's JSON model document (network.py:430-479)."""
    with open(path) as fh:
        try:
            doc = json.load(fh)
        except json.JSONDecodeError as exc:
            raise ModelFormatError(f"not a valid model document: {exc}") from exc
    for section in ("meta", "feature_norm", "params", "calibration"):
        if section not in doc:
            raise ModelFormatError(f"missing section '{section}'")
    if doc["meta"].get("format") != "pseudospec-model":
        raise ModelFormatError("missing or unknown format marker in 'meta'")

    def block(b, name, shape):
        if not isinstance(b, dict) or "shape" not in b or "data" not in b:
            raise ModelFormatError(f"field '{name}' is not a shape-prefixed array")
        if tuple(b["shape"]) != tuple(shape):
            raise ModelFormatError(f"field '{name}' has shape {b['shape']}, expected {list(shape)}")
        exp = int(np.prod(shape, dtype=int)) if shape else 1
        if len(b["data"]) != exp:
            raise ModelFormatError(f"field '{name}' holds {len(b['data'])} values, expected {exp}")
        return np.asarray(b["data"], dtype=float).reshape(shape)

    params = {k: block(doc["params"].get(k), f"params.{k}", s) for k, s in PARAM_SHAPES.items()}
    mean = block(doc["feature_norm"].get("mean"), "feature_norm.mean", (FEATURE_DIM,))
    std = block(doc["feature_norm"].get("std"), "feature_norm.std", (FEATURE_DIM,))
    if "tau_star" not in doc["calibration"]:
        raise ModelFormatError("missing field 'calibration.tau_star'")
    tau = doc["calibration"]["tau_star"]
    meta = {k: v for k, v in doc["meta"].items() if k not in ("format", "version")}
    return ModelBundle(params, mean, std, None if tau is None else float(tau), meta)


def load_npz(path) -> ModelBundle:
    z = np.load(path)
    return ModelBundle({k: z[k] for k in PARAM_SHAPES}, z["feature_mean"], z["feature_std"],
                       float(z["tau_star"]) if "tau_star" in z else None)


# ----------------------------------------------------------------------------- features
EPS = 1e-12
LOG_CAP = 16.0
PROBE_DELTAS = (0.5, 1.0, 2.0)


@dataclass
class GlobalFeatures:
    values: np.ndarray   # (30,)
    eigvals: np.ndarray  # (n,) complex
    singvals: np.ndarray


def _capped_log10(x: float) -> float:
    if not np.isfinite(x) or x <= 0:
        return LOG_CAP
    return float(min(np.log10(x), LOG_CAP))


def _resolvent_ratio(A, centroid, delta, seed) -> float:
    rng = np.random.default_rng(np.random.PCG64(seed))
    b = rng.standard_normal(A.shape[0])
    z = complex(centroid) + delta
    try:
        x = np.linalg.solve(z * np.eye(A.shape[0]) - A, b.astype(complex))
    except np.linalg.LinAlgError:
        return LOG_CAP
    return _capped_log10(float(np.linalg.norm(x) / np.linalg.norm(b)))


class _Blas1:
    """OpenBLAS pinned to one thread while any feature computation runs (reference-counted: the BLAS
    thread count is process-global, so concurrent prefetch threads must not restore it under each other)."""

    def __init__(self):
        self._lock = threading.Lock()
        self._depth = 0
        self._ctx = None

    def __enter__(self):
        with self._lock:
            if self._depth == 0:
                from threadpoolctl import threadpool_limits
                self._ctx = threadpool_limits(1)
            self._depth += 1

    def __exit__(self, *exc):
        with self._lock:
            self._depth -= 1
            if self._depth == 0:
                self._ctx.restore_original_limits()
                self._ctx = None


_BLAS1 = _Blas1()
_FEAT_LOCK = threading.Lock()
_FEAT: "OrderedDict[tuple, Future]" = OrderedDict()  # (matrix digest, probe_seed) -> Future[GlobalFeatures]
_FEAT_MAX = 64
_FEAT_POOL: ThreadPoolExecutor | None = None


def _feat_key(A, probe_seed: int) -> tuple:
    if isinstance(A, core.BandMatrix):
        data, shape = A.band, ("band", A.kl, A.ku, A.n)
    else:
        data = np.ascontiguousarray(np.asarray(A))
        shape = data.shape
    return (shape, str(data.dtype), hashlib.blake2b(data.tobytes(), digest_size=16).digest(), int(probe_seed))


def _compute_features(A, probe_seed: int) -> GlobalFeatures:
    with _BLAS1:
        return _global_features(A, probe_seed)


def global_features(A, probe_seed: int = 0) -> GlobalFeatures:
    """f1..f30 per matrix (restates features.py:63-117 operation for operation; host LAPACK).

    LAPACK runs pinned to one BLAS thread: eig of a non-normal matrix changes bits with the
    OpenBLAS thread count, and the reference's benchmark protocol is single-thread
    (cli.py:168-172), so this makes the features reproducible on any host.

    O(n^3) per matrix (eig, two SVDs, three solves) and a pure function of (A, probe_seed), so results
    are cached per (matrix contents, seed): a matrix whose features were prefetched
    (prefetch_global_features, on host threads while the GPU sweeps) or computed before is not
    recomputed. SURVEY 8(f) row 1."""
    key = _feat_key(A, probe_seed)
    with _FEAT_LOCK:
        fut = _FEAT.get(key)
        if fut is not None:
            _FEAT.move_to_end(key)
    if fut is None:
        gf = _compute_features(A, probe_seed)
        fut = Future()
        fut.set_result(gf)
        with _FEAT_LOCK:
            _FEAT[key] = fut
            while len(_FEAT) > _FEAT_MAX:
                _FEAT.popitem(last=False)
        return gf
    return fut.result()


def prefetch_global_features(items, workers: int | None = None) -> int:
    """Start computing global_features for (A, probe_seed) pairs on host threads (one BLAS thread each),
    so they overlap the GPU sweeps and each other; global_features() then returns the prefetched value.
    Returns the number of computations started."""
    global _FEAT_POOL
    started = 0
    with _FEAT_LOCK:
        if _FEAT_POOL is None:
            n = workers or max(1, (os.cpu_count() or 2) - 1)
            _FEAT_POOL = ThreadPoolExecutor(max_workers=n, thread_name_prefix="psb-features")
        for A, seed in items:
            key = _feat_key(A, seed)
            if key in _FEAT:
                continue
            _FEAT[key] = _FEAT_POOL.submit(_compute_features, A, int(seed))
            started += 1
        while len(_FEAT) > _FEAT_MAX:
            _FEAT.popitem(last=False)
    return started


def clear_feature_cache():
    with _FEAT_LOCK:
        _FEAT.clear()


def _global_features(A, probe_seed: int) -> GlobalFeatures:
    if isinstance(A, core.BandMatrix):
        A = A.todense()
    A = core.require_matrix(A)
    if np.iscomplexobj(A) and np.all(A.imag == 0):
        A = A.real.copy()
    fro = float(np.linalg.norm(A, "fro"))
    A_tilde = A / (fro + EPS)
    lam, V = np.linalg.eig(A)
    sv = np.linalg.svd(A, compute_uv=False)
    re, im, mod = lam.real, lam.imag, np.abs(lam)
    f = np.empty(30)
    f[0], f[1], f[2], f[3] = re.mean(), re.std(), re.min(), re.max()
    f[4], f[5], f[6], f[7] = im.mean(), im.std(), im.min(), im.max()
    f[8], f[9] = mod.max(), mod.min()
    f[10] = np.linalg.norm(A - A.T, "fro") / (fro + EPS)
    f[11] = np.linalg.norm(A - A.conj().T, "fro") / (fro + EPS)
    kappa = np.inf if sv[-1] == 0 else sv[0] / sv[-1]
    f[12] = _capped_log10(kappa + EPS)
    f[13] = sv[0] / (fro + EPS)
    f[14] = np.abs(A).sum(axis=0).max() / (fro + EPS)
    f[15] = np.abs(A).sum(axis=1).max() / (fro + EPS)
    d = np.abs(np.diag(A))
    f[16], f[17] = d.mean(), d.std()
    off = np.abs(A - np.diag(np.diag(A)))
    f[18], f[19] = off.mean(), off.std()
    f[20] = np.mean(np.abs(A) > 1e-10)
    sq = np.abs(A_tilde) ** 2 if np.iscomplexobj(A_tilde) else A_tilde ** 2
    f[21], f[22] = sq.mean(), sq.std()
    sv_V = np.linalg.svd(V, compute_uv=False)
    kappa_V = np.inf if sv_V[-1] == 0 else sv_V[0] / sv_V[-1]
    f[23] = _capped_log10(kappa_V + EPS)
    f[24] = np.log10(np.linalg.norm(A - A.conj().T, "fro") / (fro + EPS) + EPS)
    f[25] = (sv[0] - sv[-1]) / (sv[0] + EPS)
    f[26] = (mod.max() - mod.min()) / (mod.max() + EPS)
    centroid = complex(lam.mean())
    for k, delta in enumerate(PROBE_DELTAS):
        f[27 + k] = _resolvent_ratio(A, centroid, delta, mix64(probe_seed, k))
    return GlobalFeatures(values=f, eigvals=lam, singvals=sv)


# ----------------------------------------------------------------------------- K2 calls
def _predict_points(bundle: ModelBundle, gf: GlobalFeatures, zs: np.ndarray) -> np.ndarray:
    """Network probability at each z (pipeline.py:169-172) on the K2 kernel."""
    zs = np.ascontiguousarray(np.asarray(zs, dtype=complex).ravel())
    eig = np.ascontiguousarray(np.asarray(gf.eigvals, dtype=complex))
    emean = np.array([eig.mean()], dtype=complex)  # numpy's reduction order, as features.py:135
    params = bundle.packed()
    prob = np.empty(zs.size)
    if zs.size == 0:
        return prob
    h = _lib.handle()
    with h.lock:
        rc = h.lib.psb_predict_points(h.h, _lib._ptr(params), _lib._ptr(bundle.feature_mean),
                                      _lib._ptr(bundle.feature_std), _lib._ptr(np.ascontiguousarray(gf.values)),
                                      _lib._ptr(eig), eig.size, _lib._ptr(emean), _lib._ptr(zs), zs.size,
                                      _lib._ptr(prob))
    if rc != _lib.PSB_OK:
        raise ParameterError(h.error()) if rc == _lib.PSB_ERR_PARAM else RuntimeError(h.error())
    return prob


def predict_map(bundle: ModelBundle, A, grid: ComplexGrid, probe_seed: int = 0) -> np.ndarray:
    gf = global_features(A, probe_seed=probe_seed)
    return _predict_points(bundle, gf, grid.points().ravel()).reshape(grid.shape)


def _fine_points(flagged: np.ndarray, ay, ax, stride: int, ny: int, nx: int):
    """Row/col indices of every non-anchor point of every flagged s x s cell, in the reference's
    order (pipeline.py:206-215: cells in np.nonzero order, points row-major within a cell, clipped at
    the grid border). Vectorised: one (cells, s*s - 1) offset table, filtered in place (order kept)."""
    iy, ix = np.nonzero(flagged)
    if iy.size == 0:
        return np.zeros(0, int), np.zeros(0, int)
    dr, dc = np.divmod(np.arange(1, stride * stride), stride)  # row-major within a cell, anchor excluded
    rr = (np.asarray(ay)[iy][:, None] + dr[None, :]).ravel()
    cc = (np.asarray(ax)[ix][:, None] + dc[None, :]).ravel()
    keep = (rr < ny) & (cc < nx)
    return rr[keep], cc[keep]


def _fine_points_loop(flagged: np.ndarray, ay, ax, stride: int, ny: int, nx: int):
    """The per-cell loop _fine_points replaces (kept as the test's reference for the order)."""
    rows, cols = [], []
    for iy, ix in zip(*np.nonzero(flagged)):
        r0, c0 = ay[iy], ax[ix]
        rr, cc = np.meshgrid(np.arange(r0, min(r0 + stride, ny)), np.arange(c0, min(c0 + stride, nx)),
                             indexing="ij")
        rr, cc = rr.ravel(), cc.ravel()
        keep = ~((rr == r0) & (cc == c0))
        rows.append(rr[keep])
        cols.append(cc[keep])
    if not rows:
        return np.zeros(0, int), np.zeros(0, int)
    return np.concatenate(rows), np.concatenate(cols)


def hierarchical_predict(bundle: ModelBundle, A, grid: ComplexGrid, stride: int = 4, probe_seed: int = 0,
                         gf: GlobalFeatures | None = None):
    """Coarse-to-fine probability field (pipeline.py:182-224); returns (prob, n_evals)."""
    if stride < 2:
        raise ParameterError(f"stride must be >= 2, got {stride}")
    if gf is None:
        gf = global_features(A, probe_seed=probe_seed)
    points = grid.points()
    ay = np.arange(0, grid.ny, stride)
    ax = np.arange(0, grid.nx, stride)
    coarse_pts = points[np.ix_(ay, ax)]
    p_coarse = _predict_points(bundle, gf, coarse_pts.ravel()).reshape(coarse_pts.shape)
    tau_coarse = np.percentile(p_coarse, 80)
    flagged = p_coarse >= tau_coarse
    prob = np.zeros(grid.shape)
    prob[np.ix_(ay, ax)] = np.where(flagged, p_coarse, 0.0)
    rows, cols = _fine_points(flagged, ay, ax, stride, grid.ny, grid.nx)
    n_evals = p_coarse.size
    if rows.size:
        prob[rows, cols] = _predict_points(bundle, gf, points[rows, cols])
        n_evals += rows.size
    return prob, n_evals


def predicted_region(prob_field: np.ndarray, tau: float) -> np.ndarray:
    """dilate(prob >= tau, 5) (pipeline.py:227-231) on the K2 region kernel."""
    if not 0 < tau < 1:
        raise ParameterError(f"tau must lie in (0, 1), got {tau}")
    prob = np.ascontiguousarray(np.asarray(prob_field, dtype=float))
    ny, nx = prob.shape
    region = np.empty((ny, nx), dtype=np.uint8)
    cnt = C.c_int64(0)
    h = _lib.handle()
    with h.lock:
        rc = h.lib.psb_region_select(h.h, _lib._ptr(prob), ny, nx, float(tau), PRED_DILATION, _lib._ptr(region),
                                     None, C.byref(cnt))
    if rc != _lib.PSB_OK:
        raise RuntimeError(h.error())
    return region.astype(bool)


def recall_sweep(prob_field: np.ndarray, truth_dil: np.ndarray, taus=CAL_TAUS,
                 k: int = PRED_DILATION) -> np.ndarray:
    """[_recall(dilate(prob >= t, k), truth_dil) for t in taus] (pipeline.py:234-238,258-259) in
    one K2 kernel: the dilated mask at a pixel is (window max of prob) >= t."""
    prob = np.ascontiguousarray(np.asarray(prob_field, dtype=float))
    truth = np.ascontiguousarray(np.asarray(truth_dil, dtype=bool), dtype=np.uint8)
    if prob.shape != truth.shape or prob.ndim != 2:
        raise ParameterError(f"prob {prob.shape} and truth {truth.shape} must be equal 2-D shapes")
    taus = np.ascontiguousarray(np.asarray(taus, dtype=float).ravel())
    out = np.empty(taus.size)
    ny, nx = prob.shape
    h = _lib.handle()
    with h.lock:
        rc = h.lib.psb_recall_sweep(h.h, _lib._ptr(prob), _lib._ptr(truth), ny, nx, int(k), _lib._ptr(taus),
                                    taus.size, _lib._ptr(out))
    if rc != _lib.PSB_OK:
        raise RuntimeError(h.error())
    return out


@dataclass
class CalibrationReport:
    taus: np.ndarray
    median_recall: np.ndarray
    p10_recall: np.ndarray
    tau_star: float | None
    passed: bool
    recalls: np.ndarray = field(repr=False, default=None)  # (n_matrices, n_taus)


def calibrate_threshold(bundle: ModelBundle, val_corpus, grid: ComplexGrid, eps: float,
                        workers: int = 1) -> CalibrationReport:
    """Smallest tau with median validation recall >= 0.90 and 10th-percentile recall >= 0.75
    (pipeline.py:241-270). Per matrix: the exact σ map (K1), the dense probability map (K2) and
    all 90 recalls (one K2 kernel). `workers` is accepted for signature compatibility."""
    if not val_corpus:
        raise ParameterError("validation corpus is empty")
    recalls = np.empty((len(val_corpus), CAL_TAUS.size))
    # host features of every matrix start now, on host threads, and overlap the GPU σ maps below
    prefetch_global_features([(e.matrix, e.probe_seed) for e in val_corpus])
    for row, entry in enumerate(val_corpus):
        fld = core.full_pseudospectrum(entry.matrix, grid, label=f"matrix {entry.index}")
        truth_dil = core.dilate(core.sensitive_zone(fld, eps), TRUTH_DILATION)
        pmap = predict_map(bundle, entry.matrix, grid, probe_seed=entry.probe_seed)
        recalls[row] = recall_sweep(pmap, truth_dil, CAL_TAUS, PRED_DILATION)
    med = np.median(recalls, axis=0)
    p10 = np.percentile(recalls, 10, axis=0)
    passing = (med >= 0.90) & (p10 >= 0.75)
    if passing.any():
        best = int(np.argmax(passing))
        return CalibrationReport(CAL_TAUS.copy(), med, p10, tau_star=float(CAL_TAUS[best]), passed=True,
                                 recalls=recalls)
    return CalibrationReport(CAL_TAUS.copy(), med, p10, tau_star=None, passed=False, recalls=recalls)


@dataclass
class HybridResult:
    field: SigmaField
    region: np.ndarray
    prob_field: np.ndarray
    t_nn: float
    t_restricted: float
    nn_evaluations: int


def hybrid_pseudospectrum(bundle: ModelBundle, A, grid: ComplexGrid, eps: float, probe_seed: int = 0,
                          stride: int = 4, label: str = "matrix") -> HybridResult:
    """Predict the sensitive region (K2), then σ_min only there (K1) (pipeline.py:273-297)."""
    if bundle.tau_star is None:
        raise ParameterError("model bundle carries no calibrated threshold")
    if eps <= 0:
        raise ParameterError(f"eps must be positive, got {eps}")
    t0 = time.perf_counter()
    prob, n_evals = hierarchical_predict(bundle, A, grid, stride=stride, probe_seed=probe_seed)
    region = predicted_region(prob, bundle.tau_star)  # K2 region; its index list stays on the device
    t_nn = time.perf_counter() - t0
    t0 = time.perf_counter()
    if region.any():  # restricted_field on the device-side selection (no region upload, no host compaction)
        fld = SigmaField(grid, core._selection_call(A, grid, region, label))
    else:
        fld = SigmaField(grid, np.full(grid.shape, np.nan))
    t_restricted = time.perf_counter() - t0
    fld.eps = eps
    return HybridResult(field=fld, region=region, prob_field=prob, t_nn=t_nn, t_restricted=t_restricted,
                        nn_evaluations=n_evals)
