"""C5 batch cost model (development tool, one B200): for every matrix, the engine split on a coarse subgrid
(core.engine_split, every `stride`-th grid point each way) next to the full map's device time and engine
counts. Fits time ~ a * nB_sub + b * nL_sub + c and reports how well the subgrid split predicts the cost
(the LPT order of shard.dynamic_matrix_batch). Writes gpurun_out/c5_costmodel.json.

Usage: python tools/c5_costmodel.py [stride, default 16]
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2605_04550_b200 import configs, core  # noqa: E402

stride = int(sys.argv[1]) if len(sys.argv) > 1 else 16
cfg = configs.CONFIGS["C5"]
pts = cfg.grid.points()
sub = np.ascontiguousarray(pts[::stride, ::stride].ravel())
rows = []
for m in range(cfg.batch):
    A = cfg.matrix(m)
    core.full_pseudospectrum(A, cfg.grid)
    st = core.last_stats()
    t0 = time.perf_counter()
    nb, nl = core.engine_split(A, sub)
    t_est = time.perf_counter() - t0
    est = core.last_stats()
    rows.append({"m": m, "ms": st["ms_total"], "n_bisect": st["n_bisect"], "n_lanczos": st["n_lanczos"],
                 "ms_bisect": st["ms_bisect"], "ms_lanczos": st["ms_lanczos"], "sub_bisect": nb, "sub_lanczos": nl,
                 "est_ms_device": est["ms_classify"], "est_s_wall": t_est})
    print(rows[-1], flush=True)
t = np.array([r["ms"] for r in rows])
X = np.array([[r["sub_bisect"], r["sub_lanczos"], 1.0] for r in rows])
coef, *_ = np.linalg.lstsq(X, t, rcond=None)
pred = X @ coef
print("fit ms ~ %.4g nB_sub + %.4g nL_sub + %.4g; rank corr %.3f; rel err median %.2f max %.2f" % (
    *coef, np.corrcoef(np.argsort(np.argsort(t)), np.argsort(np.argsort(pred)))[0, 1],
    np.median(np.abs(pred - t) / t), np.max(np.abs(pred - t) / t)))
os.makedirs("gpurun_out", exist_ok=True)
with open("gpurun_out/c5_costmodel.json", "w") as f:
    json.dump({"stride": stride, "rows": rows, "coef": coef.tolist()}, f)
