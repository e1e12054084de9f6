import sys, numpy as np
sys.path.insert(0, '.')
from paper_2605_04550_b200 import core, configs, _lib
from oracle.sigma_oracle import smin_restated
cfg = configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
A = cfg.matrix(); Ad = A.todense().real
pts = cfg.grid.points()
v, it, st = core.smin_many(A, pts.ravel(), return_info=True)
v = v.reshape(cfg.grid.shape); it = it.reshape(cfg.grid.shape); st = st.reshape(cfg.grid.shape)
dx = cfg.grid.xs()[1] - cfg.grid.xs()[0]
bad = np.argwhere(np.abs(np.diff(v, axis=1)) > dx * (1 + 1e-9) + 1e-12)
print("violations", len(bad))
cand = set()
for i, j in bad[:20]:
    cand.add((i, j)); cand.add((i, j + 1))
cand = sorted(cand)[:24]
zs = np.array([pts[i, j] for i, j in cand])
want = smin_restated(Ad, zs)
for (i, j), w in zip(cand, want):
    print(i, j, pts[i, j], "got", v[i, j], "want", w, "rel", abs(v[i, j] - w) / w, "st", st[i, j], "it", it[i, j])
