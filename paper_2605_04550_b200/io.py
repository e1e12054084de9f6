"""Drop-in for the field / mask writers of `pseudospec.io` (io.py:92-115).

The reference formats one f-string per grid point in a Python loop; here the rows are
formatted by libpsb200.so's host writers (csrc/psb_io.cpp) on all host threads and the file
bytes are identical: same header, row-major order, every float as f"{v:.17g}". log10 of the
field is taken with numpy exactly as the reference does (io.py:97-98), so the third column
carries the same bits.
"""

from __future__ import annotations

import os

import numpy as np

from . import _lib
from .core import ComplexGrid, ParameterError, SigmaField


def _check(rc: int, path) -> None:
    if rc == _lib.PSB_ERR_IO:
        raise OSError(f"could not write {path}")
    if rc != _lib.PSB_OK:
        raise ParameterError(f"bad writer arguments for {path}")


def write_field_csv(path, field: SigmaField, nthreads: int = 0) -> None:
    """Rows `x,y,log10_smin` in row-major grid order; unevaluated points emit `nan`."""
    xs = np.ascontiguousarray(field.grid.xs(), dtype=float)
    ys = np.ascontiguousarray(field.grid.ys(), dtype=float)
    with np.errstate(divide="ignore", invalid="ignore"):
        logs = np.ascontiguousarray(np.log10(field.values), dtype=float)
    lib = _lib.load_library()
    _check(lib.psb_write_field_csv(os.fsencode(path), _lib._ptr(xs), xs.size, _lib._ptr(ys), ys.size,
                                   _lib._ptr(logs), int(nthreads)), path)


def write_mask_csv(path, mask: np.ndarray, grid: ComplexGrid, nthreads: int = 0) -> None:
    """Rows `x,y,flag` with flag in {0,1}, row-major grid order."""
    mask = np.asarray(mask, dtype=bool)
    if mask.shape != grid.shape:
        raise ParameterError(f"mask shape {mask.shape} does not match grid {grid.shape}")
    xs = np.ascontiguousarray(grid.xs(), dtype=float)
    ys = np.ascontiguousarray(grid.ys(), dtype=float)
    m = np.ascontiguousarray(mask, dtype=np.uint8)
    lib = _lib.load_library()
    _check(lib.psb_write_mask_csv(os.fsencode(path), _lib._ptr(xs), xs.size, _lib._ptr(ys), ys.size,
                                  _lib._ptr(m), int(nthreads)), path)
