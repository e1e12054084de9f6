"""A/B two library builds on full σ maps (development tool): bitwise equality and per-matrix kernel times.

Usage: python tools/ab_maps.py C5 0,1,17,63 ablib/libpsb200_base.so paper_2605_04550_b200/libpsb200.so
A side may carry environment knobs: lib.so@PSB_SEQ=1,PSB_TAU=2e-3
"""
import json
import os
import subprocess
import sys

import numpy as np

name, mats, la, lb = sys.argv[1], [int(m) for m in sys.argv[2].split(",")], sys.argv[3], sys.argv[4]
code = r"""
import json, sys, numpy as np
sys.path.insert(0, '.')
from paper_2605_04550_b200 import configs, core
c = configs.CONFIGS[sys.argv[1]]
out = {}
for m in [int(x) for x in sys.argv[2].split(',')]:
    A = c.matrix(m)
    core.full_pseudospectrum(A, c.grid)          # warm (upload, launch shapes)
    best = None
    for _ in range(2):
        f = core.full_pseudospectrum(A, c.grid)
        st = core.last_stats()
        if best is None or st['ms_total'] < best['ms_total']:
            best = st
    np.save(f'/tmp/ab_{sys.argv[3]}_{m}.npy', f.values)
    out[m] = {k: best[k] for k in ('ms_total', 'ms_bisect', 'ms_lanczos', 'ms_classify', 'n_bisect', 'n_lanczos')}
print(json.dumps(out))
"""
res = {}
for tag, spec in (("a", la), ("b", lb)):
    lib, _, knobs = spec.partition("@")
    extra = dict(kv.split("=", 1) for kv in knobs.split(",") if kv)
    r = subprocess.run([sys.executable, "-c", code, name, sys.argv[2], tag], capture_output=True, text=True,
                       env={**os.environ, "PSB200_LIB": lib, **extra})
    if r.returncode:
        print(r.stderr[-3000:])
        sys.exit(1)
    res[tag] = json.loads(r.stdout.strip().splitlines()[-1])
for m in mats:
    a, b = np.load(f"/tmp/ab_a_{m}.npy"), np.load(f"/tmp/ab_b_{m}.npy")
    eq = np.array_equal(a, b)
    relmax = np.max(np.abs(a - b) / np.maximum(np.abs(a), 1e-300))
    nd = int(np.sum(a != b))
    dabs = float(np.max(np.abs(a - b))) / max(float(np.max(a)), 1e-300)  # largest change against the map's scale
    if nd:
        sys.path.insert(0, '.')
        from paper_2605_04550_b200 import configs
        A = configs.CONFIGS[name].matrix(m)
        if hasattr(A, "band"):  # band[d + kl, i] = A[i, i + d]: column i + d
            c2 = np.zeros(A.n)
            for d in range(-A.kl, A.ku + 1):
                i = np.arange(max(0, -d), min(A.n, A.n - d))
                c2[i + d] += np.abs(A.band[d + A.kl, i]) ** 2
            cmax = float(np.sqrt(c2.max()))
        else:
            cmax = float(np.max(np.linalg.norm(np.asarray(A), axis=0)))
        dm = a != b
        print(f"  changed points: max |diff| / max_j ||A e_j|| = {np.max(np.abs(a - b)[dm]) / cmax:.2e}, "
              f"A-side values there <= {np.max(a[dm]) / cmax:.2e} ||A e_j||, B-side <= {np.max(b[dm]) / cmax:.2e}")
    if nd:
        rel = np.abs(a - b) / np.maximum(np.abs(a), 1e-300)
        k = int(np.nanargmax(rel))
        print(f"  largest relative change at flat index {k}: A {a.ravel()[k]:.6e}  B {b.ravel()[k]:.6e}")
    ta, tb = res["a"][str(m)], res["b"][str(m)]
    print(f"{name} m={m}: bitwise {eq} (max rel {relmax:.2e}, {nd} differ, max|diff|/max {dabs:.1e}) | A total {ta['ms_total']:.1f} B {ta['ms_bisect']:.1f} "
          f"L {ta['ms_lanczos']:.1f} C {ta.get('ms_classify', 0):.1f} | B total {tb['ms_total']:.1f} "
          f"B {tb['ms_bisect']:.1f} L {tb['ms_lanczos']:.1f} C {tb.get('ms_classify', 0):.1f} ms")
