"""ctypes binding of libpsb200.so (include/psb200.h).

This is the reference-side binding a maintainer would add to `pseudospec` (see
INTEGRATION.md): plain pointers and sizes, numpy arrays passed by address, the GIL released
for the duration of every call. There is deliberately no Python fallback: if the shared
library or a CUDA device is missing, `handle()` raises `BackendUnavailable` and nothing is
computed.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("PSB200_LIB", _HERE / "libpsb200.so"))

PSB_OK, PSB_ERR_PARAM, PSB_ERR_NUMERICAL, PSB_ERR_CUDA, PSB_ERR_IO = 0, 1, 2, 3, 4

#: every symbol include/psb200.h declares (checked by the CPU test-suite)
EXPORTS = (
    "psb_create", "psb_destroy", "psb_last_error", "psb_version", "psb_set_matrix",
    "psb_smin_points", "psb_smin_grid", "psb_smin_points_device", "psb_engine_split", "psb_get_stats",
    "psb_predict_points", "psb_region_select", "psb_smin_selection", "psb_fp64_peak", "psb_recall_sweep",
    "psb_write_field_csv", "psb_write_mask_csv",
)


class BackendUnavailable(RuntimeError):
    """libpsb200.so could not be loaded or no CUDA device is visible."""


class Opts(C.Structure):
    _fields_ = [("tau", C.c_double), ("bis_rtol", C.c_double), ("kmax", C.c_int32),
                ("force_engine", C.c_int32), ("refill", C.c_int32), ("reserved", C.c_int32)]


class Stats(C.Structure):
    _fields_ = [("n_points", C.c_int64), ("n_lanczos", C.c_int64), ("n_bisect", C.c_int64),
                ("lanczos_iters", C.c_int64), ("pd_tests", C.c_int64),
                ("flops_bisect", C.c_double), ("flops_lanczos", C.c_double),
                ("bytes_lanczos", C.c_double), ("ms_bisect", C.c_double),
                ("ms_lanczos", C.c_double), ("ms_total", C.c_double),
                ("grid_bisect", C.c_int32), ("grid_lanczos", C.c_int32),
                ("ms_classify", C.c_double), ("flops_classify", C.c_double), ("ms_fallback", C.c_double),
                ("launches", C.c_int32), ("reserved", C.c_int32)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


_P = C.c_void_p
_lib = None
_lib_lock = threading.Lock()


def load_library(path: Path | str | None = None) -> C.CDLL:
    """Load and type the shared library (no GPU needed for this step)."""
    global _lib
    with _lib_lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path is not None else LIB_PATH
        if not p.exists():
            raise BackendUnavailable(
                f"{p} not found; build it with `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = C.CDLL(str(p))
        lib.psb_create.argtypes = [C.c_int, C.POINTER(_P)]
        lib.psb_destroy.argtypes = [_P]
        lib.psb_destroy.restype = None
        lib.psb_last_error.argtypes = [_P]
        lib.psb_last_error.restype = C.c_char_p
        lib.psb_version.argtypes = []
        lib.psb_set_matrix.argtypes = [_P, _P, C.c_int32, C.c_int32, C.c_int32]
        lib.psb_smin_points.argtypes = [_P, _P, C.c_int64, C.POINTER(Opts), _P, _P, _P,
                                        C.POINTER(C.c_int64)]
        lib.psb_smin_selection.argtypes = [_P, _P, C.c_int32, _P, C.c_int32, C.POINTER(Opts), _P, _P, _P,
                                           C.POINTER(C.c_int64)]
        lib.psb_smin_grid.argtypes = [_P, _P, C.c_int32, _P, C.c_int32, _P, C.POINTER(Opts), _P, _P,
                                      _P, C.POINTER(C.c_int64)]
        lib.psb_smin_points_device.argtypes = [_P, _P, C.c_int64, C.POINTER(Opts), _P, _P, _P, _P]
        lib.psb_engine_split.argtypes = [_P, _P, C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        lib.psb_get_stats.argtypes = [_P, C.POINTER(Stats)]
        lib.psb_fp64_peak.argtypes = [_P, C.POINTER(C.c_double)]
        lib.psb_recall_sweep.argtypes = [_P, _P, _P, C.c_int32, C.c_int32, C.c_int32, _P, C.c_int32, _P]
        lib.psb_write_field_csv.argtypes = [C.c_char_p, _P, C.c_int64, _P, C.c_int64, _P, C.c_int32]
        lib.psb_write_mask_csv.argtypes = [C.c_char_p, _P, C.c_int64, _P, C.c_int64, _P, C.c_int32]
        lib.psb_predict_points.argtypes = [_P, _P, _P, _P, _P, _P, C.c_int32, _P, _P, C.c_int64, _P]
        lib.psb_region_select.argtypes = [_P, _P, C.c_int32, C.c_int32, C.c_double, C.c_int32, _P, _P,
                                          C.POINTER(C.c_int64)]
        if path is None:
            _lib = lib
        return lib


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(_P)


class Handle:
    """One device context of the library (one per process and device)."""

    def __init__(self, device: int = 0):
        self.lib = load_library()
        h = _P()
        rc = self.lib.psb_create(int(device), C.byref(h))
        if rc != PSB_OK or not h:
            raise BackendUnavailable(f"psb_create(device={device}) failed with code {rc} "
                                     "(no CUDA device visible?)")
        self.h = h
        self.device = device
        self.lock = threading.Lock()
        self._matrix_key = None

    def close(self):
        if getattr(self, "h", None):
            self.lib.psb_destroy(self.h)
            self.h = None

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass

    def error(self) -> str:
        return self.lib.psb_last_error(self.h).decode()

    def fp64_peak(self) -> float:
        """Measured DFMA throughput of the device, TFLOP/s."""
        t = C.c_double(0.0)
        rc = self.lib.psb_fp64_peak(self.h, C.byref(t))
        if rc != PSB_OK:
            raise RuntimeError(f"psb_fp64_peak failed: {self.error()}")
        return t.value

    def stats(self) -> dict:
        s = Stats()
        self.lib.psb_get_stats(self.h, C.byref(s))
        return s.as_dict()


_handles: dict[int, Handle] = {}


def default_device() -> int:
    """The caller's device: $PSB200_DEVICE, else torch's current device when torch has already
    initialised CUDA in this process (a torch.distributed rank bound with torch.cuda.set_device),
    else $LOCAL_RANK (one process per GPU under torchrun), else 0."""
    env = os.environ.get("PSB200_DEVICE")
    if env is not None:
        return int(env)
    import sys
    torch = sys.modules.get("torch")
    if torch is not None:
        try:
            if torch.cuda.is_initialized():
                return int(torch.cuda.current_device())
        except Exception:
            pass
    return int(os.environ.get("LOCAL_RANK", "0"))


def handle(device: int | None = None) -> Handle:
    """Process-wide handle for `device` (default: `default_device()`)."""
    if device is None:
        device = default_device()
    with _lib_lock:
        h = _handles.get(device)
    if h is None:
        h = Handle(device)
        with _lib_lock:
            _handles[device] = h
    return h


def make_opts(tau=None, bis_rtol=None, kmax=None, force_engine=0, refill=None) -> Opts:
    o = Opts()
    o.tau = float(tau) if tau else 0.0
    o.bis_rtol = float(bis_rtol) if bis_rtol else 0.0
    o.kmax = int(kmax) if kmax else 0
    o.force_engine = int(force_engine)
    o.refill = int(refill) if refill else 0
    return o
