"""One σ sweep of a config through the device API (for ncu / compute-sanitizer runs)."""
import sys, ctypes as C
import numpy as np
sys.path.insert(0, '.')
from paper_2605_04550_b200 import _lib, configs, core

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cfg = configs.CONFIGS[name]
A = cfg.matrix(0)
pts = np.ascontiguousarray(cfg.grid.points().ravel())
for r in range(reps):
    s = core.smin_many(A, pts)
st = core.last_stats()
print(name, {k: st[k] for k in ("n_lanczos", "n_bisect", "lanczos_iters", "pd_tests", "ms_bisect", "ms_lanczos")})
