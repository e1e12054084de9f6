import sys, numpy as np
sys.path.insert(0, '.')
from paper_2605_04550_b200 import configs, core
for name in ("C2", "C3"):
    cfg = configs.CONFIGS[name]
    A = cfg.matrix(0) if name != "C2" else cfg.matrix()
    pts = cfg.grid.points().ravel()
    v, it, st = core.smin_many(A, pts, return_info=True)
    b = st == 1
    S = np.abs(pts[b]) + core.last_stats().get("anorm", 0) if False else None
    h = core._lib.handle() if hasattr(core, "_lib") else None
    # anorm = sqrt(|A|_1 |A|_inf) as psb_set_matrix
    Ad = A.todense() if hasattr(A, "todense") else A
    anorm = np.sqrt(np.abs(Ad).sum(0).max() * np.abs(Ad).sum(1).max())
    lam0 = (3e-3 * (np.abs(pts[b]) + anorm)) ** 2
    ratio = v[b] ** 2 / lam0
    srch = np.ceil(np.log(ratio) / np.log(16))
    rounds = (it[b] - 1) / 2
    print(name, "bisect pts", b.sum(), "tests/pt mean", it[b].mean(), "p50", np.median(it[b]), "p90", np.percentile(it[b], 90),
          "max", it[b].max(), "| est search rounds mean", srch.mean(), "| rounds mean", rounds.mean(),
          "| sigma/(tauS) p50", np.median(np.sqrt(ratio)), "p90", np.percentile(np.sqrt(ratio), 90))
    print("  rounds hist", np.bincount(rounds.astype(int))[:40])
