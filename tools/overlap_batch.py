"""Matrix-batch pipelining experiment (development tool, one B200): S host threads, each with its own library
handle (own streams and buffers), pull C5 matrices from a shared queue, so one matrix's kernel tail overlaps
the next matrix's start. Prints the batch's wall time per S and checks the maps are bitwise equal to S = 1.

Usage: python tools/overlap_batch.py [matrices, default 0-15] [S values, default 1,2,3]
"""
import ctypes as C
import queue
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2605_04550_b200 import _lib, configs, core  # noqa: E402

cfg = configs.CONFIGS["C5"]
mats = [int(m) for m in sys.argv[1].split(",")] if len(sys.argv) > 1 else list(range(16))
svals = [int(s) for s in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 2, 3]
zs = np.ascontiguousarray(cfg.grid.points().ravel())
P = zs.size
d_zs = torch.from_numpy(zs.view(np.float64)).cuda()
bands = {m: core.as_band(cfg.matrix(m)) for m in mats}
outs = {m: torch.empty(P, dtype=torch.float64, device="cuda") for m in mats}
handles = [_lib.Handle(0) for _ in range(max(svals))]


def run(h, m):
    core._set_matrix(h, bands[m])
    rc = h.lib.psb_smin_points_device(h.h, C.c_void_p(d_zs.data_ptr()), P, None, C.c_void_p(outs[m].data_ptr()),
                                      None, None, None)
    assert rc == 0, h.error()


def batch(S):
    q = queue.Queue()
    for m in mats:
        q.put(m)

    def worker(h):
        while True:
            try:
                m = q.get_nowait()
            except queue.Empty:
                return
            run(h, m)

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    th = [threading.Thread(target=worker, args=(handles[i],)) for i in range(S)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    torch.cuda.synchronize()
    return time.perf_counter() - t0


for h in handles:  # warm every handle (launch shapes, buffers)
    run(h, mats[0])
ref = None
for S in svals:
    t = batch(S)
    t2 = batch(S)
    maps = {m: outs[m].cpu().numpy().copy() for m in mats}
    if ref is None:
        ref = maps
    same = all(np.array_equal(maps[m], ref[m]) for m in mats)
    print(f"S={S}: batch of {len(mats)} matrices {min(t, t2) * 1e3:.0f} ms "
          f"({len(mats) * P / min(t, t2) / 1e6:.2f} M points/s), bitwise equal to S=1: {same}", flush=True)
