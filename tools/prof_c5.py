"""One full σ map of a config's matrix (profiling driver for ncu / PSB_PROF; development tool).

Usage: python tools/prof_c5.py [config] [matrix]      e.g.  ncu -k regex:k_lanczos -c 1 ... tools/prof_c5.py C5 1
"""
import sys

sys.path.insert(0, ".")
from paper_2605_04550_b200 import configs, core  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
m = int(sys.argv[2]) if len(sys.argv) > 2 else 1
c = configs.CONFIGS[name]
f = core.full_pseudospectrum(c.matrix(m), c.grid)
print(name, m, {k: round(v, 2) if isinstance(v, float) else v for k, v in core.last_stats().items()})
