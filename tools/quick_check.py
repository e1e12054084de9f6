"""Quick GPU-vs-oracle check used during development (run under gpurun)."""
import sys, time, json
import numpy as np
sys.path.insert(0, '.')
from paper_2605_04550_b200 import core, configs, _lib
from oracle.sigma_oracle import smin_restated, floored_rel_err


def check(name, A, zs, opts=None):
    t = time.time()
    got, it, st = core.smin_many(A, zs, opts=opts, return_info=True)
    tg = time.time() - t
    stats = core.last_stats()
    Ad = A.todense() if isinstance(A, core.BandMatrix) else A
    t = time.time()
    want = smin_restated(Ad, zs)
    to = time.time() - t
    floor = 1e-5 * np.linalg.norm(Ad, 2)
    e = floored_rel_err(got, want, floor)
    print(json.dumps(dict(name=name, P=len(zs), max_err=float(e.max()), n_bad=int((e > 1e-9).sum()),
                          gpu_s=round(tg, 4), oracle_s=round(to, 2),
                          engines=dict(L=int((st == 0).sum()), B=int((st == 1).sum()), sing=int((st == 2).sum())),
                          it_L_mean=float(it[st == 0].mean()) if (st == 0).any() else 0,
                          it_B_mean=float(it[st == 1].mean()) if (st == 1).any() else 0,
                          ms_B=stats['ms_bisect'], ms_L=stats['ms_lanczos'])), flush=True)
    if e.max() > 1e-9:
        b = np.argsort(e)[-5:]
        for i in b:
            print("   worst", zs[i], got[i], want[i], e[i], it[i], st[i])
    return e


which = sys.argv[1:] or ["C1", "C2", "C3", "C4"]
rng = np.random.default_rng(0)
for w in which:
    cfg = configs.CONFIGS[w]
    A = cfg.matrix(0)
    npts = {"C1": 2500, "C2": 300, "C3": 48, "C4": 12, "C5": 2}[w]
    idx, zs = configs.sample_points(cfg, npts, 123)
    check(w, A, zs)
    if w in ("C1", "C2"):
        for fe in ((1, 2) if w == "C1" else (1,)):
            check(f"{w}-force{fe}", A, zs[:200], opts=_lib.make_opts(force_engine=fe))
# small dense/banded random (reference acceptance c01 style)
worst = 0
for t in range(20):
    n = int(rng.integers(4, 17)); beta = int(rng.integers(1, min(4, n - 1) + 1))
    A = rng.integers(-1, 2, size=(n, n)).astype(float)
    i = np.arange(n); A[np.abs(i[:, None] - i[None, :]) > beta] = 0
    zs = rng.uniform(-4, 4, 30) + 1j * rng.uniform(-4, 4, 30)
    got = core.smin_many(A, zs)
    want = smin_restated(A, zs)
    worst = max(worst, float((np.abs(got - want) / np.maximum(1.0, want)).max()))
print("small random worst rel(1,want)", worst)
M = rng.standard_normal((12, 12)); A = (M + M.T) / 2
lam = np.linalg.eigvalsh(A)
zs = core.make_grid(-3, 3, -3, 3, 10, 10).points().ravel()
d = np.abs(zs[:, None] - lam[None, :]).min(axis=1)
print("normality worst", float(np.abs(core.smin_many(A, zs) - d).max()))
g = core.make_grid(-4, 4, -4, 4, 20, 20)
Ad = configs.grcar_band(30).todense()
full = core.full_pseudospectrum(Ad, g)
reg = np.zeros(g.shape, bool); reg[3:9, 5:17] = True
rf = core.restricted_field(Ad, g, reg)
print("restricted==full bitwise", bool(np.array_equal(rf.values[reg], full.values[reg])), "nan off", bool(np.isnan(rf.values[~reg]).all()))
pts = g.points()
print("pointwise==batched", all(core.smin_at(Ad, pts[i, j]) == full.values[i, j] for i in range(0, 20, 3) for j in range(0, 20, 3)))
