"""Drop-in for `pseudospec.core` (reference: pkg/src/pseudospec/core.py).

Same names, argument meaning and error behaviour as the reference module; every sigma_min
value comes from the CUDA engines in libpsb200.so through the C ABI (`_lib.py`). There is no
CPU path: without the library or a GPU the σ functions raise `BackendUnavailable`.

Differences from the reference, each deliberate:
  * complex A is accepted (the reference silently casts to real, core.py:112-119; configs
    C3/C5 of BASELINE.json are complex), and A must be banded with kl, ku <= 16;
  * `workers` is accepted and ignored (one process drives the GPU; core.py:186-195 used a
    process pool), `chunk` likewise (values are chunk-invariant, core.py:148-149);
  * σ_min agrees with the reference's zgesdd to the parity gate in DESIGN.md
    (|Δ| <= 1e-9 * max(σ_ref, 1e-5 ||A||_2)), not bitwise; restricted == full, worker and
    chunk invariance, and batched == pointwise hold bitwise, as in the reference.
"""

from __future__ import annotations

import ctypes as C
import hashlib
from dataclasses import dataclass

import numpy as np

from . import _lib


class ParameterError(ValueError):
    """Invalid argument to a public operation (core.py:18-19)."""


class NumericalError(ArithmeticError):
    """A σ_min evaluation failed (core.py:22-23)."""


class GenerationError(RuntimeError):
    """Matrix generation exhausted its rejection budget (core.py:26-27)."""


class CalibrationError(RuntimeError):
    """Threshold calibration found no admissible threshold (core.py:30-31)."""


class ModelFormatError(ValueError):
    """A model file is missing fields or carries malformed arrays (core.py:34-35)."""


@dataclass(frozen=True)
class ComplexGrid:
    """Uniform grid; point (i, j) is x[j] + 1j*y[i] (core.py:38-78)."""

    x_min: float
    x_max: float
    y_min: float
    y_max: float
    nx: int
    ny: int

    def __post_init__(self):
        if not (self.x_min < self.x_max and self.y_min < self.y_max):
            raise ParameterError(
                f"grid bounds must be ordered, got x=[{self.x_min}, {self.x_max}] "
                f"y=[{self.y_min}, {self.y_max}]")
        if self.nx < 2 or self.ny < 2:
            raise ParameterError(f"need nx, ny >= 2, got nx={self.nx} ny={self.ny}")

    @property
    def shape(self) -> tuple[int, int]:
        return (self.ny, self.nx)

    @property
    def size(self) -> int:
        return self.nx * self.ny

    def xs(self) -> np.ndarray:
        return np.linspace(self.x_min, self.x_max, self.nx)

    def ys(self) -> np.ndarray:
        return np.linspace(self.y_min, self.y_max, self.ny)

    def points(self) -> np.ndarray:
        return self.xs()[None, :] + 1j * self.ys()[:, None]


def make_grid(x_min, x_max, y_min, y_max, nx, ny) -> ComplexGrid:
    return ComplexGrid(float(x_min), float(x_max), float(y_min), float(y_max), int(nx), int(ny))


@dataclass
class SigmaField:
    """Per-grid-point σ_min values; NaN marks unevaluated points (core.py:86-109)."""

    grid: ComplexGrid
    values: np.ndarray
    eps: float | None = None

    def __post_init__(self):
        self.values = np.asarray(self.values, dtype=float)
        if self.values.shape != self.grid.shape:
            raise ParameterError(
                f"field shape {self.values.shape} does not match grid {self.grid.shape}")

    def evaluated(self) -> np.ndarray:
        return ~np.isnan(self.values)

    def mask(self, eps: float) -> np.ndarray:
        if eps <= 0:
            raise ParameterError(f"eps must be positive, got {eps}")
        with np.errstate(invalid="ignore"):
            return np.asarray(self.values <= eps)


# ------------------------------------------------------------------ matrices and bands

def require_matrix(A) -> np.ndarray:
    """Validate A as a finite square matrix, n >= 2 (core.py:112-119), keeping complex."""
    A = np.asarray(A)
    A = A.astype(complex if np.iscomplexobj(A) else float, copy=False)
    if A.ndim != 2 or A.shape[0] != A.shape[1] or A.shape[0] < 2:
        raise ParameterError(f"expected a square matrix with n >= 2, got shape {A.shape}")
    if not np.all(np.isfinite(A)):
        raise ParameterError("matrix entries must be finite")
    return A


def bandwidths(A: np.ndarray) -> tuple[int, int]:
    """(kl, ku): largest sub- and super-diagonal offsets holding a nonzero."""
    r, c = np.nonzero(A)
    if r.size == 0:
        return 0, 0
    return int(max(0, (r - c).max())), int(max(0, (c - r).max()))


def band_of(A: np.ndarray, kl: int | None = None, ku: int | None = None) -> np.ndarray:
    """Diagonal-major band: band[d + kl, i] = A[i, i + d] (include/psb200.h layout)."""
    A = np.asarray(A)
    n = A.shape[0]
    if kl is None or ku is None:
        kl, ku = bandwidths(A)
    band = np.zeros((kl + ku + 1, n), dtype=complex)
    for d in range(-kl, ku + 1):
        diag = np.diagonal(A, offset=d)
        lo = max(0, -d)
        band[d + kl, lo:lo + diag.size] = diag
    return band


class BandMatrix:
    """A banded matrix given directly by its diagonals (no dense n x n copy).

    `band[d + kl, i] = A[i, i + d]`; entries whose column falls outside [0, n) are ignored.
    Accepted everywhere a dense A is (BASELINE C5 uses n = 4000 bands)."""

    def __init__(self, band: np.ndarray, kl: int, ku: int):
        band = np.ascontiguousarray(np.asarray(band, dtype=complex))
        if band.ndim != 2 or band.shape[0] != kl + ku + 1:
            raise ParameterError(f"band must have shape ({kl + ku + 1}, n), got {band.shape}")
        self.band, self.kl, self.ku, self.n = band, int(kl), int(ku), band.shape[1]
        if self.n < 2:
            raise ParameterError(f"expected a square matrix with n >= 2, got n={self.n}")
        if not np.all(np.isfinite(band)):
            raise ParameterError("matrix entries must be finite")
        for d in range(-kl, ku + 1):  # canonical zeros outside the matrix
            if d < 0:
                self.band[d + kl, :-d] = 0
            elif d > 0:
                self.band[d + kl, self.n - d:] = 0

    @property
    def shape(self):
        return (self.n, self.n)

    def todense(self) -> np.ndarray:
        A = np.zeros((self.n, self.n), dtype=complex)
        for d in range(-self.kl, self.ku + 1):
            lo = max(0, -d)
            m = self.n - abs(d)
            A[np.arange(lo, lo + m), np.arange(lo, lo + m) + d] = self.band[d + self.kl, lo:lo + m]
        return A


MAX_BAND = 16


def as_band(A):
    """(band, kl, ku, n) for a dense array or a BandMatrix; kl, ku <= MAX_BAND."""
    if isinstance(A, BandMatrix):
        band, kl, ku, n = A.band, A.kl, A.ku, A.n
    else:
        A = require_matrix(A)
        kl, ku = bandwidths(A)
        band, n = np.ascontiguousarray(band_of(A, kl, ku)), A.shape[0]
    if kl > MAX_BAND or ku > MAX_BAND:
        raise ParameterError(f"band evaluator supports kl, ku <= {MAX_BAND}, got kl={kl} ku={ku}")
    return band, kl, ku, n


def _set_matrix(h: _lib.Handle, A):
    band, kl, ku, n = A if isinstance(A, tuple) else as_band(A)
    if kl > 16 or ku > 16:
        raise ParameterError(f"band evaluator supports kl, ku <= 16, got kl={kl} ku={ku}")
    key = (n, kl, ku, hashlib.blake2b(band.tobytes(), digest_size=16).digest())
    if h._matrix_key == key:
        return n
    h._matrix_key = None  # a failed upload leaves no matrix the key could vouch for
    rc = h.lib.psb_set_matrix(h.h, band.ctypes.data_as(C.c_void_p), n, kl, ku)
    if rc == _lib.PSB_ERR_PARAM:
        raise ParameterError(h.error())
    if rc != _lib.PSB_OK:
        raise RuntimeError(f"psb_set_matrix failed ({rc}): {h.error()}")
    h._matrix_key = key
    return n


def _raise(h, rc, label, zs_flat=None, fail_index=-1):
    if rc == _lib.PSB_ERR_PARAM:
        raise ParameterError(h.error())
    if rc == _lib.PSB_ERR_NUMERICAL:
        z = zs_flat[fail_index] if zs_flat is not None and fail_index >= 0 else None
        raise NumericalError(
            f"sigma_min evaluation failed to converge on {label} at point index {fail_index}, z={z}"
            f" ({h.error()})")
    raise RuntimeError(f"libpsb200 error {rc}: {h.error()}")


def eigenvalues(A, label: str = "matrix") -> np.ndarray:
    """All n eigenvalues (core.py:122-128). Host LAPACK, as in the reference."""
    A = require_matrix(A.todense() if isinstance(A, BandMatrix) else A)
    try:
        return np.linalg.eigvals(A)
    except np.linalg.LinAlgError as exc:
        raise NumericalError(f"eigenvalue solver failed to converge on {label}") from exc


_last_stats: dict = {}


def last_stats() -> dict:
    """Engine statistics of the most recent σ call (points per engine, steps, tests, times)."""
    return dict(_last_stats)


def smin_many(A, zs: np.ndarray, label: str = "matrix", chunk: int = 512, *,
              opts: _lib.Opts | None = None, return_info: bool = False, device: int | None = None):
    """σ_min(z I - A) for a 1-D array of shift points (core.py:141-168).

    `device`: the CUDA device to run on (default `_lib.default_device()`: the rank's device
    under torch.distributed). A non-finite shift raises NumericalError naming its index and z,
    as the reference's LinAlgError path does (core.py:157-166)."""
    zs = np.ascontiguousarray(np.asarray(zs, dtype=complex).ravel())
    band = as_band(A)  # validate on the host first (ParameterError without touching the device)
    bad = np.flatnonzero(~np.isfinite(zs))
    if bad.size:
        i = int(bad[0])
        raise NumericalError(f"SVD failed to converge on {label} at point index {i}, z={zs[i]}")
    h = _lib.handle(device)
    with h.lock:
        _set_matrix(h, band)
        P = zs.size
        out = np.empty(P)
        iters = np.empty(P, dtype=np.int32)
        status = np.empty(P, dtype=np.int8)
        fi = C.c_int64(-1)
        rc = h.lib.psb_smin_points(h.h, zs.ctypes.data_as(C.c_void_p), P,
                                   C.byref(opts) if opts is not None else None,
                                   _lib._ptr(out), _lib._ptr(iters), _lib._ptr(status), C.byref(fi))
        _last_stats.clear()
        _last_stats.update(h.stats())
        if rc != _lib.PSB_OK:
            _raise(h, rc, label, zs, fi.value)
    if return_info:
        return out, iters, status
    return out


def engine_split(A, zs: np.ndarray, *, device: int | None = None) -> tuple[int, int]:
    """How many of the shifts `zs` the bisection and the Lanczos engine would take (the classification
    test alone, no σ): the cost estimate batch scheduling uses (shard.batch_cost_estimates)."""
    zs = np.ascontiguousarray(np.asarray(zs, dtype=complex).ravel())
    band = as_band(A)
    h = _lib.handle(device)
    nb, nl = C.c_int64(0), C.c_int64(0)
    with h.lock:
        _set_matrix(h, band)
        rc = h.lib.psb_engine_split(h.h, zs.ctypes.data_as(C.c_void_p), zs.size, C.byref(nb), C.byref(nl))
        if rc == _lib.PSB_ERR_PARAM:
            raise ParameterError(h.error())
        if rc != _lib.PSB_OK:
            raise RuntimeError(f"psb_engine_split failed ({rc}): {h.error()}")
    return int(nb.value), int(nl.value)


def smin_at(A, z: complex, label: str = "matrix", *, device: int | None = None) -> float:
    """σ_min of z I - A at one point (core.py:131-138); identical bits to smin_many."""
    z = complex(z)
    if not np.isfinite(z):
        raise NumericalError(f"SVD failed to converge on {label} at z={z}")
    return float(smin_many(A, np.array([z], dtype=complex), label=label, device=device)[0])


def _selection_call(A, grid: ComplexGrid, region, label, opts=None, device=None):
    """restricted_field on the selection psb_region_select left on the device (`region` is that
    selection's mask, used only to name a failing point)."""
    xs = np.ascontiguousarray(grid.xs())
    ys = np.ascontiguousarray(grid.ys())
    band = as_band(A)
    h = _lib.handle(device)
    with h.lock:
        _set_matrix(h, band)
        out = np.empty(grid.shape)
        fi = C.c_int64(-1)
        rc = h.lib.psb_smin_selection(h.h, _lib._ptr(xs), grid.nx, _lib._ptr(ys), grid.ny,
                                      C.byref(opts) if opts is not None else None, _lib._ptr(out), None, None,
                                      C.byref(fi))
        _last_stats.clear()
        _last_stats.update(h.stats())
        if rc != _lib.PSB_OK:
            pts = grid.points().ravel()[np.flatnonzero(np.asarray(region).ravel())]
            _raise(h, rc, label, pts, fi.value)
    return out


def _grid_call(A, grid: ComplexGrid, region, label, opts=None, device=None):
    xs = np.ascontiguousarray(grid.xs())
    ys = np.ascontiguousarray(grid.ys())
    band = as_band(A)
    h = _lib.handle(device)
    with h.lock:
        _set_matrix(h, band)
        out = np.empty(grid.shape)
        status = np.empty(grid.shape, dtype=np.int8)
        reg = None if region is None else np.ascontiguousarray(region, dtype=np.uint8)
        fi = C.c_int64(-1)
        rc = h.lib.psb_smin_grid(h.h, _lib._ptr(xs), grid.nx, _lib._ptr(ys), grid.ny, _lib._ptr(reg),
                                 C.byref(opts) if opts is not None else None,
                                 _lib._ptr(out), None, _lib._ptr(status), C.byref(fi))
        _last_stats.clear()
        _last_stats.update(h.stats())
        if rc != _lib.PSB_OK:
            pts = grid.points().ravel()
            if region is not None:
                pts = pts[np.flatnonzero(np.asarray(region).ravel())]
            _raise(h, rc, label, pts, fi.value)
    return out


def full_pseudospectrum(A, grid: ComplexGrid, label: str = "matrix",
                        workers: int = 1, *, opts: _lib.Opts | None = None,
                        device: int | None = None) -> SigmaField:
    """σ_min at every grid point (core.py:177-195). `workers` is ignored (one GPU process)."""
    return SigmaField(grid, _grid_call(A, grid, None, label, opts, device))


def restricted_field(A, grid: ComplexGrid, region: np.ndarray, label: str = "matrix", *,
                     opts: _lib.Opts | None = None, device: int | None = None) -> SigmaField:
    """σ_min only on the True points of `region`; the rest stays NaN (core.py:198-208)."""
    region = _check_mask(region, grid.shape)
    if not region.any():
        return SigmaField(grid, np.full(grid.shape, np.nan))
    return SigmaField(grid, _grid_call(A, grid, region, label, opts, device))


def sensitive_zone(field: SigmaField, eps: float) -> np.ndarray:
    """Evaluated points with σ_min <= eps (core.py:211-213)."""
    return field.mask(eps)


def _check_mask(mask, shape) -> np.ndarray:
    mask = np.asarray(mask)
    if mask.dtype != bool or mask.shape != tuple(shape):
        raise ParameterError(f"expected boolean mask of shape {tuple(shape)}, "
                             f"got {mask.dtype} {mask.shape}")
    return mask


def dilate(mask: np.ndarray, k: int) -> np.ndarray:
    """k x k box dilation clipped at the borders (core.py:224-231), separable max filter."""
    mask = np.asarray(mask, dtype=bool)
    if k < 1 or k % 2 == 0:
        raise ParameterError(f"structuring element size must be odd and positive, got {k}")
    if k == 1:
        return mask.copy()
    h = k // 2
    out = mask.copy()
    for axis in (0, 1):
        src = out
        acc = src.copy()
        n = src.shape[axis]
        for s in range(1, h + 1):
            if s >= n:
                break
            sl_dst = [slice(None)] * 2
            sl_src = [slice(None)] * 2
            sl_dst[axis] = slice(s, None)
            sl_src[axis] = slice(None, n - s)
            acc[tuple(sl_dst)] |= src[tuple(sl_src)]
            sl_dst[axis] = slice(None, n - s)
            sl_src[axis] = slice(s, None)
            acc[tuple(sl_dst)] |= src[tuple(sl_src)]
        out = acc
    return out
