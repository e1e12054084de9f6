"""Classification threshold tau A/B: engine mix, sweep time and the worst floored error against the
committed reference fixtures, per tau (development tool)."""
import sys, numpy as np
sys.path.insert(0, '.')
from paper_2605_04550_b200 import _lib, configs, core
from oracle.sigma_oracle import floored_rel_err

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
taus = [float(t) for t in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["3e-3", "1e-3"])]
cfg = configs.CONFIGS[name]
A = cfg.matrix()
pts = cfg.grid.points().ravel()
fx = [np.load(f"tests/golden/{name.lower()}_{s}.npz") for s in ("sample", "wide")
      if __import__("os").path.exists(f"tests/golden/{name.lower()}_{s}.npz")]
for tau in taus:
    o = _lib.make_opts(tau=tau)
    best = 1e9
    for _ in range(2):
        core.smin_many(A, pts, opts=o)
        s = core.last_stats()
        best = min(best, s["ms_total"])
    errs = []
    for d in fx:
        got = core.smin_many(A, d["zs"], opts=o)
        errs.append(floored_rel_err(got, d["sigma"], 1e-5 * float(d["norm2"])).max())
    print(f"{name} tau={tau:.1e} ms_total={best:8.2f} L={s['n_lanczos']} B={s['n_bisect']} "
          f"Lsteps={s['lanczos_iters']} tests={s['pd_tests']} ms_L={s['ms_lanczos']:.2f} ms_B={s['ms_bisect']:.2f} "
          f"worst_err={max(errs):.2e} over {sum(len(d['zs']) for d in fx)} fixture pts", flush=True)
