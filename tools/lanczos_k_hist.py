import sys, numpy as np
sys.path.insert(0, '.')
from paper_2605_04550_b200 import core, configs
cfg = configs.CONFIGS[sys.argv[1]]
v, it, st = core.smin_many(cfg.matrix(), cfg.grid.points().ravel(), return_info=True)
k = it[st == 0]
print(sys.argv[1], "lanczos steps: mean %.2f p50 %d p90 %d p99 %d max %d" % (k.mean(), np.median(k), np.percentile(k, 90), np.percentile(k, 99), k.max()))
print(" hist", np.bincount(np.minimum(k, 30)))
idx = np.flatnonzero(st.ravel() == 0)
kk = it.ravel()[idx]
w = kk[: (kk.size // 32) * 32].reshape(-1, 32)
print("  per-32-group: mean of max %.2f, mean of mean %.2f" % (w.max(1).mean(), w.mean(1).mean()))
