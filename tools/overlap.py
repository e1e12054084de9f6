"""Time each engine alone vs the combined pipeline on one config (development tool)."""
import sys, time, numpy as np
sys.path.insert(0, '.')
from paper_2605_04550_b200 import core, configs, _lib

cfg = configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
A = cfg.matrix()
pts = cfg.grid.points().ravel()
v, it, st = core.smin_many(A, pts, return_info=True)
pB, pL = pts[st == 1], pts[st == 0]


def t(zs, opts=None, reps=5):
    best = 1e9
    for _ in range(reps):
        core.smin_many(A, zs, opts=opts)
        s = core.last_stats()
        best = min(best, s["ms_total"])
    return best, s


for name, zs, o in (("all", pts, None), ("bisect-only pts", pB, None), ("lanczos-only pts", pL, None),
                    ("lanczos pts forced L", pL, _lib.make_opts(force_engine=1))):
    ms, s = t(zs, o)
    print(f"{name:22s} P={zs.size:7d} ms_total={ms:8.3f} ms_bisect={s['ms_bisect']:8.3f} ms_lanczos={s['ms_lanczos']:8.3f}")
