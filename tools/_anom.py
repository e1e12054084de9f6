import sys, numpy as np
sys.path.insert(0, '.')
from paper_2605_04550_b200 import _lib, configs, core
cases = {"C2": [-0.6180904522613065-1.9522613065326633j], "C3": [1.2969505994425892+0.5598915580565724j],
         "C4": [-923035.8469667323-64363.99217221135j, -2784778.7776908036-108277.88649706458j],
         "C5": [-0.5480134967786521+2.77254956420496j]}
out = {}
for nm, zs in cases.items():
    A = configs.CONFIGS[nm].matrix()
    zs = np.array(zs)
    # same grid point values: find exact grid points
    pts = configs.CONFIGS[nm].grid.points().ravel()
    idx = [int(np.argmin(np.abs(pts - z))) for z in zs]
    zz = pts[idx]
    for tau in (3e-3, 1e-3, 6e-4, 2.5e-4):
        v, it, st = core.smin_many(A, zz, opts=_lib.make_opts(tau=tau), return_info=True)
        print(nm, tau, v.tolist(), it.tolist(), st.tolist(), flush=True)
    out[nm] = zz
np.save("gpurun_out/anom_pts.npy", np.concatenate(list(out.values())))
