import sys, numpy as np
sys.path.insert(0, '.')
from paper_2605_04550_b200 import core, configs
cfg = configs.CONFIGS[sys.argv[1]]
v, it, st = core.smin_many(cfg.matrix(), cfg.grid.points().ravel(), return_info=True)
b = it[st == 1]
print(sys.argv[1], "bisect tests: mean %.1f p50 %d p90 %d p99 %d max %d" % (b.mean(), np.median(b), np.percentile(b, 90), np.percentile(b, 99), b.max()))
# per-warp max over consecutive groups of 32 bisect points (list order ~ grid order)
idx = np.flatnonzero(st.ravel() == 1)
bb = it.ravel()[idx]
w = bb[: (bb.size // 32) * 32].reshape(-1, 32)
print("  per-32-group: mean of max %.1f, mean of mean %.1f" % (w.max(1).mean(), w.mean(1).mean()))
