"""cProfile of hierarchical_predict on the C4 guided case (development tool)."""
import sys, cProfile, pstats, numpy as np
sys.path.insert(0, '.')
from paper_2605_04550_b200 import configs, core, pipeline
z = np.load('tests/golden/c4_guided.npz')
b4 = pipeline.load_npz('tests/golden/model_c4.npz')
S = float(z['scale'])
grid = core.make_grid(*(v * S for v in configs.C4_BOX), 512, 512)
gf = pipeline.GlobalFeatures(values=z['f30'], eigvals=z['eig'], singvals=np.zeros(0))
pipeline.hierarchical_predict(b4, None, grid, gf=gf)
cProfile.run('pipeline.hierarchical_predict(b4, None, grid, gf=gf)', '/tmp/h.prof')
pstats.Stats('/tmp/h.prof').sort_stats('cumulative').print_stats(15)
