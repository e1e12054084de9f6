"""K2 probabilities of a library build on the C4 guided points (development tool): saves them for a bitwise A/B."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2605_04550_b200 import configs, core, pipeline  # noqa: E402

z = np.load("tests/golden/c4_guided.npz")
b4 = pipeline.load_npz("tests/golden/model_c4.npz")
S = float(z["scale"])
grid = core.make_grid(*(v * S for v in configs.C4_BOX), 512, 512)
gf = pipeline.GlobalFeatures(values=z["f30"], eigvals=z["eig"], singvals=np.zeros(0))
np.save(sys.argv[1], pipeline._predict_points(b4, gf, grid.points().ravel()[::7]))
