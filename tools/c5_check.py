"""C5 (64 x n=4000 (3,3) complex, 1024^2 grid each): throughput on a strided subsample of matrix m + parity."""
import sys, time, numpy as np
sys.path.insert(0, '.')
from paper_2605_04550_b200 import core, configs
cfg = configs.CONFIGS["C5"]
m = int(sys.argv[1]) if len(sys.argv) > 1 else 0
stride = int(sys.argv[2]) if len(sys.argv) > 2 else 64
A = cfg.matrix(m)
pts = cfg.grid.points()[::stride, ::stride].ravel()
core.smin_many(A, pts[:256]); core.smin_many(A, pts)
t = time.time()
v, it, st = core.smin_many(A, pts, return_info=True)
dt = time.time() - t
s = core.last_stats()
print(f"C5 m={m} P={pts.size} wall {dt:.3f}s -> {pts.size/dt:.0f} pts/s; kernel ms {s['ms_total']:.1f} "
      f"L={s['n_lanczos']} (steps {s['lanczos_iters']}) B={s['n_bisect']} (tests {s['pd_tests']}) ms_B {s['ms_bisect']:.1f} ms_L {s['ms_lanczos']:.1f}")
z = np.load('tests/golden/c5_sample.npz')
for r, mm in enumerate(z['matrices']):
    if int(mm) == m:
        g = core.smin_many(A, z['zs'][r])
        e = np.abs(g - z['sigma'][r]) / np.maximum(z['sigma'][r], 1e-5 * z['norm2'][r])
        print("parity worst", e.max())
