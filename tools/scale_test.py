import sys, numpy as np
sys.path.insert(0, '.')
from oracle.sigma_oracle import smin_restated, floored_rel_err
from paper_2605_04550_b200 import configs, core
A0 = configs.grcar_band(60).todense().real
zs0 = core.make_grid(-1, 3, -3.5, 3.5, 7, 7).points().ravel()
for s in (1e-200, 1e-100, 1e-30, 1.0, 1e30, 1e100, 1e150, 1e200):
    A = A0 * s; zs = zs0 * s
    try:
        got, it, st = core.smin_many(A, zs, return_info=True)
        want = smin_restated(A, zs)
        e = floored_rel_err(got, want, 1e-5 * np.linalg.norm(A, 2))
        print(f"scale {s:.0e}: worst {e.max():.2e} statuses {np.bincount(st, minlength=5)[:5]}")
    except Exception as ex:
        print(f"scale {s:.0e}: {type(ex).__name__}: {str(ex)[:120]}")
