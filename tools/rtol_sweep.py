"""Bisection tolerance vs accuracy (golden fixtures) and C2/C3 step time (development tool)."""
import sys
import numpy as np
sys.path.insert(0, '.')
from paper_2605_04550_b200 import _lib, configs, core

G = "tests/golden/"
for rtol in [float(x) for x in (sys.argv[1:] or ["2e-12", "2e-11", "1e-10"])]:
    o = _lib.make_opts(bis_rtol=rtol)
    out = [f"rtol={rtol:g}"]
    for name, f in (("C1", None), ("C2", "c2_sample"), ("C3", "c3_sample"), ("C4", "c4_sample")):
        cfg = configs.CONFIGS[name]
        A = cfg.matrix(0)
        if f is None:
            z = np.load(G + "c1_full.npz")
            zs, want, nrm = cfg.grid.points().ravel(), z["values"].ravel(), float(z["norm2"])
        else:
            z = np.load(G + f + ".npz")
            zs, want, nrm = z["zs"], z["sigma"], float(z["norm2"])
        got, it, st = core.smin_many(A, zs, opts=o, return_info=True)
        e = np.abs(got - want) / np.maximum(want, 1e-5 * nrm)
        out.append(f"{name} max_err {e.max():.2e} (bisect pts {e[st == 1].max() if (st == 1).any() else 0:.2e})")
    for name in ("C2", "C3"):
        cfg = configs.CONFIGS[name]
        A = cfg.matrix(0)
        pts = cfg.grid.points().ravel()
        best = 1e9
        for _ in range(4):
            core.smin_many(A, pts, opts=o)
            best = min(best, core.last_stats()["ms_total"])
        s = core.last_stats()
        out.append(f"{name} {best:.3f} ms (tests/pt {s['pd_tests'] / max(1, s['n_bisect']):.1f})")
    print(" | ".join(out), flush=True)
