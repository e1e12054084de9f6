"""Paper-scale label generation: the reference's own build_dataset over a
seeded n=64 corpus on a 100x100 grid, with σ on the B200 (shim) vs the reference's CPU path
(timed on one matrix, one BLAS thread). Development tool; prints one JSON line."""
import json
import sys
import time
from pathlib import Path

import numpy as np
from threadpoolctl import threadpool_limits

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
import pseudospec as ps  # noqa: E402

from paper_2605_04550_b200 import shim  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 16
t = time.perf_counter()
corpus = ps.generate_corpus(ps.GenSpec(n=64, seed=303), count)
t_gen = time.perf_counter() - t
grid = ps.make_grid(-4, 4, -4, 4, 100, 100)
with threadpool_limits(1):
    t = time.perf_counter()
    ref1 = ps.pipeline.build_dataset(corpus[:1], grid, eps=1e-2, seed=7)
    t_cpu1 = time.perf_counter() - t
shim.install(ps)
try:
    ps.pipeline.build_dataset(corpus[:1], grid, eps=1e-2, seed=7)  # warm-up (CUDA context, matrix upload)
    with threadpool_limits(1):
        t = time.perf_counter()
        ds = ps.pipeline.build_dataset(corpus, grid, eps=1e-2, seed=7)
        t_gpu = time.perf_counter() - t
        g1 = ps.pipeline.build_dataset(corpus[:1], grid, eps=1e-2, seed=7)
finally:
    shim.uninstall()
same = all(np.array_equal(getattr(g1, k), getattr(ref1, k)) for k in ("xy", "features", "labels", "matrix_ids"))
print(json.dumps({"matrices": count, "grid": "100x100", "sigma_evals": count * grid.size, "samples": len(ds),
                  "t_generate_s": t_gen, "t_build_dataset_gpu_s": t_gpu,
                  "sigma_evals_per_s_gpu": count * grid.size / t_gpu,
                  "t_build_dataset_cpu_1matrix_s": t_cpu1, "cpu_sigma_evals_per_s": grid.size / t_cpu1,
                  "speedup_per_matrix": t_cpu1 / (t_gpu / count), "first_matrix_identical": same}))
