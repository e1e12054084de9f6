"""Which bisection points take the most PD tests (the engine's kernel time tracks the max when
points ~ threads) — development tool."""
import sys, numpy as np
sys.path.insert(0, '.')
from paper_2605_04550_b200 import _lib, configs, core
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = configs.CONFIGS[name]
A = cfg.matrix(); Ad = A.todense()
pts = cfg.grid.points().ravel()
v, it, st = core.smin_many(A, pts, return_info=True)
dg = np.diag(Ad); c0 = 0.5 * (dg.real.min() + dg.real.max()) + 0.5j * (dg.imag.min() + dg.imag.max())
T = np.sqrt((np.abs(pts - c0) + np.abs(dg - c0).max()) ** 2 + (np.abs(Ad - np.diag(dg)) ** 2).sum(0).max())
b = st == 1
print(name, "bisection points", b.sum(), "tests: mean %.1f p50 %d p99 %d max %d" % (it[b].mean(), *np.percentile(it[b], [50, 99]), it[b].max()))
r = v / T
for lo, hi in ((0, 1e-3), (1e-3, 3e-3), (3e-3, 1e-2), (1e-2, 3e-2), (3e-2, 0.1), (0.1, 0.3), (0.3, 2)):
    m = b & (r >= lo) & (r < hi)
    if m.any(): print(f"  r in [{lo:g},{hi:g}): {m.sum():6d} pts, tests mean {it[m].mean():.1f} max {it[m].max()}")
for i in np.argsort(-np.where(b, it, 0))[:6]:
    print("   tests", it[i], "r %.3e" % r[i], "z", pts[i], "sigma %.6e" % v[i])
