import sys, time, numpy as np, ctypes as C
sys.path.insert(0, '.')
import torch
from paper_2605_04550_b200 import _lib, configs, core
cfg = configs.CONFIGS["C2"]; A = cfg.matrix(); g = cfg.grid
core.full_pseudospectrum(A, g)
def tm(f, n=20):
    ts = []
    for _ in range(n):
        torch.cuda.synchronize(); t = time.perf_counter(); f(); torch.cuda.synchronize(); ts.append((time.perf_counter() - t) * 1e3)
    return np.median(ts), np.min(ts)
print("full_pseudospectrum", tm(lambda: core.full_pseudospectrum(A, g)))
h = _lib.handle()
xs = np.ascontiguousarray(g.xs()); ys = np.ascontiguousarray(g.ys()); out = np.empty(g.shape); st = np.empty(g.shape, np.int8); fi = C.c_int64(-1)
def raw():
    h.lib.psb_smin_grid(h.h, _lib._ptr(xs), g.nx, _lib._ptr(ys), g.ny, None, None, _lib._ptr(out), None, _lib._ptr(st), C.byref(fi))
print("raw psb_smin_grid", tm(raw))
zs = torch.tensor(g.points().ravel()).view(torch.float64).cuda(); sig = torch.empty(g.size, dtype=torch.float64, device="cuda")
print(core.last_stats())
