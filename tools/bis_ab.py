"""Bisection-engine cost on a fixed point set (development A/B between library builds, selected
with PSB200_LIB): C2 points far from the split, forced through engine B."""
import sys, numpy as np
sys.path.insert(0, '.')
from paper_2605_04550_b200 import _lib, configs, core

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = configs.CONFIGS[name]
A = cfg.matrix()
pts = cfg.grid.points().ravel()
v = core.smin_many(A, pts)
sel = pts[v >= 0.01 * (np.abs(pts) + np.abs(A.todense()).sum(0).max())]
best = 1e9
for _ in range(5):
    core.smin_many(A, sel, opts=_lib.make_opts(force_engine=2))
    s = core.last_stats()
    best = min(best, s["ms_bisect"])
print(f"{name}: {sel.size} pts forced B: ms_bisect {best:.3f} tests {s['pd_tests']}")
_, it, st = core.smin_many(A, sel, opts=_lib.make_opts(force_engine=2), return_info=True)
print("   tests/pt: mean %.1f p50 %d p90 %d p99 %d max %d" % (it.mean(), *np.percentile(it, [50, 90, 99]), it.max()))
