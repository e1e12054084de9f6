"""C5 multi-GPU balance model (development tool, one B200): device time of every matrix of the batch, and of
every rank's share under the cyclic point deal for N = 2, 4, 8 (point p -> rank p mod N, shard.py).

No rank waits on another in either scheme (no data-path collective), so a rank's step time on N GPUs is its
own share's device time; this measures each share alone on one GPU and models the N-GPU step as the max
over ranks. Writes gpurun_out/c5_balance.json.

Usage: python tools/c5_balance.py [matrices, default 0-63]
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2605_04550_b200 import configs, core  # noqa: E402

cfg = configs.CONFIGS["C5"]
mats = [int(m) for m in sys.argv[1].split(",")] if len(sys.argv) > 1 else list(range(64))
zs = cfg.grid.points().ravel()
out = {"full": {}, "share": {}}


def dev_ms(A, pts):
    core.smin_many(A, pts)
    return core.last_stats()["ms_total"]


for m in mats:
    A = cfg.matrix(m)
    core.full_pseudospectrum(A, cfg.grid)  # upload + launch shapes
    out["full"][m] = dev_ms(A, zs)
    for N in (2, 4, 8):
        out["share"].setdefault(N, {})[m] = [dev_ms(A, zs[r::N]) for r in range(N)]
    print(m, round(out["full"][m], 1), {N: [round(x, 1) for x in out["share"][N][m]] for N in (2, 4, 8)}, flush=True)

os.makedirs("gpurun_out", exist_ok=True)
with open("gpurun_out/c5_balance.json", "w") as f:
    json.dump(out, f)
