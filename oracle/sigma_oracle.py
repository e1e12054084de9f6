"""ORACLE (test infrastructure only) — CPU restatement of pseudospec.core.smin_many.

Follows pkg/src/pseudospec/core.py:141-168 exactly: for each shift z, the dense matrix
z*I - A is formed (core.py:154) and its smallest singular value is the last entry of
np.linalg.svd(..., compute_uv=False) (core.py:156,167), i.e. LAPACK zgesdd through numpy's
_umath_linalg.svd gufunc (numpy 2.3.5, bundled OpenBLAS 0.3.30). The only change is that
complex A is *not* cast to real (core.py:112-119 `require_real_matrix` would drop the
imaginary part of BASELINE configs C3/C5); for real A the bits equal the reference's
(pinned by tests/test_oracle.py against fixtures produced by the reference itself).

BLAS is pinned to one thread: the reference's bits depend on the OpenBLAS thread count
(SURVEY.md §0.3), and the shipped golden (demos/output_01_field.csv) was produced single-thread.
"""

from __future__ import annotations

import numpy as np
from threadpoolctl import threadpool_limits


def smin_restated(A, zs, chunk: int = 1, threads: int = 1) -> np.ndarray:
    """σ_min(z I - A) for every z in zs (core.py:141-168 without the real cast). BLAS runs on `threads`
    threads (1 by default: the fixtures' bits; the reference's protocol is single-thread)."""
    A = np.asarray(A)
    A = A.astype(complex if np.iscomplexobj(A) else float)
    zs = np.asarray(zs, dtype=complex).ravel()
    n = A.shape[0]
    eye = np.eye(n)
    out = np.empty(zs.size)
    with threadpool_limits(threads):
        for start in range(0, zs.size, chunk):
            zc = zs[start:start + chunk]
            shifted = zc[:, None, None] * eye - A
            out[start:start + chunk] = np.linalg.svd(shifted, compute_uv=False)[:, -1]
    return out


def smin_gesvd(A, zs) -> np.ndarray:
    """Independent route (QR-based gesvd driver), as tests/test_core.py:82-85 of the reference."""
    import scipy.linalg
    A = np.asarray(A)
    n = A.shape[0]
    with threadpool_limits(1):
        return np.array([scipy.linalg.svd(z * np.eye(n) - A, compute_uv=False, lapack_driver="gesvd")[-1]
                         for z in np.asarray(zs, dtype=complex).ravel()])


def parity_floor(A) -> float:
    """σ_floor = 1e-5 * ||A||_2 of the floored parity gate."""
    A = np.asarray(A)
    return 1e-5 * float(np.linalg.norm(A, 2))


def floored_rel_err(got, want, floor) -> np.ndarray:
    """|Δ| / max(σ_ref, floor): the parity metric (bound 1e-9)."""
    got = np.asarray(got, dtype=float)
    want = np.asarray(want, dtype=float)
    return np.abs(got - want) / np.maximum(want, floor)
