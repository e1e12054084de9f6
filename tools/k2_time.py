import sys, time, numpy as np
sys.path.insert(0, '.')
from paper_2605_04550_b200 import configs, core, pipeline
z = np.load('tests/golden/c4_guided.npz')
b4 = pipeline.load_npz('tests/golden/model_c4.npz')
S = float(z['scale'])
grid = core.make_grid(*(v * S for v in configs.C4_BOX), 512, 512)
gf = pipeline.GlobalFeatures(values=z['f30'], eigvals=z['eig'], singvals=np.zeros(0))
zs = grid.points().ravel()[:65536]
pipeline._predict_points(b4, gf, zs[:1024])
for P in (4096, 65536):
    t = time.perf_counter(); pipeline._predict_points(b4, gf, zs[:P]); dt = time.perf_counter() - t
    print('K2', P, 'points', dt * 1e3, 'ms')
t = time.perf_counter(); prob, ne = pipeline.hierarchical_predict(b4, None, grid, gf=gf); dt = time.perf_counter() - t
print('hierarchical', dt * 1e3, 'ms', ne)
t = time.perf_counter(); r = pipeline.predicted_region(prob, b4.tau_star); dt = time.perf_counter() - t
print('region', dt * 1e3, 'ms')
