"""Dump full C5 σ maps (σ, engine status, iterations) of selected matrices for fixture stratification.

Usage (GPU box): python tools/c5_maps.py 0 1 17 63  -> gpurun_out/c5_maps.npz
"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2605_04550_b200 import configs, core  # noqa: E402

cfg = configs.CONFIGS["C5"]
ms = [int(a) for a in sys.argv[1:]] or [0, 1, 17, 63]
out = {}
for m in ms:
    A = cfg.matrix(m)
    t = time.time()
    xs, ys = cfg.grid.xs(), cfg.grid.ys()
    import ctypes as C
    from paper_2605_04550_b200 import _lib
    h = _lib.handle()
    with h.lock:
        core._set_matrix(h, A)
        sig = np.empty(cfg.grid.shape)
        it = np.empty(cfg.grid.shape, dtype=np.int32)
        st = np.empty(cfg.grid.shape, dtype=np.int8)
        fi = C.c_int64(-1)
        rc = h.lib.psb_smin_grid(h.h, _lib._ptr(xs), cfg.grid.nx, _lib._ptr(ys), cfg.grid.ny, None, None,
                                 _lib._ptr(sig), _lib._ptr(it), _lib._ptr(st), C.byref(fi))
    print(m, "rc", rc, "s", time.time() - t, core.last_stats() if False else h.stats(), flush=True)
    out[f"sigma_{m}"] = sig.astype(np.float32)
    out[f"status_{m}"] = st
    out[f"iters_{m}"] = it.astype(np.int16)
np.savez_compressed("gpurun_out/c5_maps.npz", matrices=np.array(ms), **out)
