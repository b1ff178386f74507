"""One 64-source eccentricity pass (target for ncu launch lists)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2404_17101_b200 as pg  # noqa: E402

dg = pg.make_config(sys.argv[1] if len(sys.argv) > 1 else "c4")
src = np.random.default_rng(0).integers(0, dg.n, 64).tolist()
torch.cuda.synchronize()
t0 = time.perf_counter()
e = pg.eccentricities(dg, src)
print("max ecc", max(e), "time", time.perf_counter() - t0)
