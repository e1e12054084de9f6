"""Bitwise comparison of two library builds on a config's full grid (development tool)."""
import os, subprocess, sys, numpy as np
sys.path.insert(0, '.')
name, la, lb = sys.argv[1], sys.argv[2], sys.argv[3]
code = ("import sys, numpy as np; sys.path.insert(0,'.'); from paper_2605_04550_b200 import configs, core; "
        f"c=configs.CONFIGS['{name}']; v=core.smin_many(c.matrix(), c.grid.points().ravel()); np.save(sys.argv[1], v)")
for lib, out in ((la, "/tmp/a.npy"), (lb, "/tmp/b.npy")):
    subprocess.run([sys.executable, "-c", code, out], check=True, env={**os.environ, "PSB200_LIB": lib})
a, b = np.load("/tmp/a.npy"), np.load("/tmp/b.npy")
print(name, "bitwise equal:", np.array_equal(a, b), "max rel diff %.2e" % np.max(np.abs(a - b) / np.maximum(a, 1e-300)))
