import sys, numpy as np
sys.path.insert(0, '.')
from paper_2605_04550_b200 import core, configs, _lib
cfg = configs.CONFIGS[sys.argv[1]]
A = cfg.matrix(); pts = cfg.grid.points().ravel()
v, it, st = core.smin_many(A, pts, return_info=True)
pL = pts[st == 0]
for R in (1, 2, 4, 8, 16, 24, 32):
    best = 1e9
    for _ in range(2):
        core.smin_many(A, pL, opts=_lib.make_opts(refill=R))
        best = min(best, core.last_stats()["ms_lanczos"])
    print(f"refill {R:2d}: lanczos ms {best:.2f}")
