"""Bisection termination tolerance A/B: kernel time, tests and fixture error per rtol (development tool)."""
import sys, os, numpy as np
sys.path.insert(0, '.')
from paper_2605_04550_b200 import _lib, configs, core
from oracle.sigma_oracle import floored_rel_err
name = sys.argv[1]
cfg = configs.CONFIGS[name]
A = cfg.matrix()
pts = cfg.grid.points().ravel()
fx = [np.load(f"tests/golden/{name.lower()}_{s}.npz") for s in ("sample", "wide") if os.path.exists(f"tests/golden/{name.lower()}_{s}.npz")]
base = None
for rt in [float(x) for x in sys.argv[2].split(",")]:
    o = _lib.make_opts(bis_rtol=rt)
    best = 1e9
    for _ in range(3):
        v, it, st = core.smin_many(A, pts, opts=o, return_info=True)
        s = core.last_stats(); best = min(best, s["ms_total"])
    if base is None: base = v
    errs = [floored_rel_err(core.smin_many(A, d["zs"], opts=o), d["sigma"], 1e-5 * float(d["norm2"])).max() for d in fx if "matrices" not in d]
    b = st == 1
    print(f"{name} rtol={rt:.0e} ms={best:.3f} ms_B={s['ms_bisect']:.3f} tests={s['pd_tests']} max_tests={it[b].max()} "
          f"fixture_err={max(errs) if errs else float('nan'):.2e} vs_first_max={np.max(np.abs(v - base) / base):.2e}", flush=True)
