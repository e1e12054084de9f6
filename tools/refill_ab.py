"""Lanczos lane-refill threshold A/B and step-count histogram on one config (development tool)."""
import sys, numpy as np
sys.path.insert(0, '.')
from paper_2605_04550_b200 import _lib, configs, core

cfg = configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
A = cfg.matrix()
pts = cfg.grid.points().ravel()
v, it, st = core.smin_many(A, pts, return_info=True)
k = it[st == 0]
q = np.percentile(k, [50, 90, 99, 99.9])
print(cfg.name if hasattr(cfg, "name") else sys.argv[1], "lanczos steps: mean %.2f p50 %d p90 %d p99 %d p99.9 %d max %d" % (k.mean(), *q, k.max()))
print(" share of lane-steps from points with k>20: %.3f, k>50: %.3f" % (k[k > 20].sum() / k.sum(), k[k > 50].sum() / k.sum()))
print(" hist", np.bincount(np.minimum(k, 40)).tolist())
for rf in [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["1", "4", "8", "16", "24"])]:
    best = 1e9
    for _ in range(2):
        core.smin_many(A, pts, opts=_lib.make_opts(refill=rf))
        best = min(best, core.last_stats()["ms_lanczos"])
    print(f" refill={rf:2d} ms_lanczos={best:.2f}", flush=True)
