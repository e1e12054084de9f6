"""Small sweeps for compute-sanitizer (memcheck / racecheck): C1 grid, a C5-shape slice, a dense
runtime-shape matrix and the two-launch engine-B path on a C4-shape grid subset."""
import sys, numpy as np
sys.path.insert(0, '.')
from paper_2605_04550_b200 import configs, core
for name, k in (("C1", 1), ("C2", 7), ("C5", 997)):
    cfg = configs.CONFIGS[name]
    v = core.smin_many(cfg.matrix(), cfg.grid.points().ravel()[::k])
    print(name, v.size, float(np.nanmax(v)), core.last_stats()["grid_bisect"], flush=True)
d = np.random.default_rng(3).standard_normal((24, 24))
print("dense", core.smin_many(d, np.array([0.3 + 0.1j, -2 + 1j]))[:2])
