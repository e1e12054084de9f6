"""Full-grid error of the bisection engine near the classification threshold: for every point that
moves from engine L (tau=1e-2) to engine B at a lower tau, compare the two results. Engine L is
accurate there (C1-C4 fixtures: <= 1e-11), so this measures engine B's squared-form error as a
function of r = sigma/S over whole grids, with c = err * 2 r^2 / eps the empirical rounding
constant (development tool)."""
import sys, numpy as np
sys.path.insert(0, '.')
from paper_2605_04550_b200 import _lib, configs, core

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
taus = [float(t) for t in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["1e-3", "6e-4", "4e-4"])]
cfg = configs.CONFIGS[name]
A = cfg.matrix()
pts = cfg.grid.points().ravel()
h = _lib.handle()
TAU_REF = 1e-2
ref, it0, st0 = core.smin_many(A, pts, opts=_lib.make_opts(tau=TAU_REF), return_info=True)
Ad = A.todense()
dg = np.diag(Ad)
c0 = 0.5 * (dg.real.min() + dg.real.max()) + 0.5j * (dg.imag.min() + dg.imag.max())
r0 = np.abs(dg - c0).max()
offsq = (np.abs(Ad - np.diag(dg)) ** 2).sum(0).max()
S = np.sqrt((np.abs(pts - c0) + r0) ** 2 + offsq)  # the engine split's scale T(z)
for tau in taus:
    v, it, st = core.smin_many(A, pts, opts=_lib.make_opts(tau=tau), return_info=True)
    moved = np.flatnonzero((st0 == 0) & (st == 1))
    e = np.abs(v[moved] - ref[moved]) / ref[moved]
    r = ref[moved] / S[moved]
    c = e * 2 * r * r / 2.22e-16
    print(f"{name} tau={tau:.1e}: {moved.size} moved; max err {e.max():.2e}; c: p50 {np.median(c):.2f} p99 {np.percentile(c, 99):.2f} max {c.max():.1f}")
    for i in np.argsort(-e)[:3]:
        print(f"   err {e[i]:.2e} r {r[i]:.2e} c {c[i]:.1f} bis_tests {it[moved[i]]} lanczos_k {it0[moved[i]]} z {pts[moved[i]]}")
