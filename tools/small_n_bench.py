"""Paper-scale workload timing (development tool): random banded n = 64 matrices (beta = 1..4, entries
in {-1, 0, 1} like the reference's generator) on a 100x100 grid, sigma_min per point."""
import sys, time, numpy as np
sys.path.insert(0, '.')
from paper_2605_04550_b200 import core
rng = np.random.default_rng(5)
g = core.make_grid(-4, 4, -4, 4, 100, 100)
pts = g.points().ravel()
for beta in (1, 2, 3, 4):
    A = np.zeros((64, 64))
    for d in range(-beta, beta + 1):
        A += np.diag(rng.integers(-1, 2, 64 - abs(d)).astype(float), d)
    core.smin_many(A, pts)
    ts = []
    for _ in range(5):
        t = time.perf_counter(); core.smin_many(A, pts); ts.append(time.perf_counter() - t)
    s = core.last_stats()
    print(f"beta={beta}: {min(ts) * 1e3:.3f} ms for {pts.size} points (L={s['n_lanczos']} B={s['n_bisect']})", flush=True)
