"""Time estimate_diameter (1000 samples, 64 sources per device pass) on BASELINE configs."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2404_17101_b200 as pg  # noqa: E402

for name in sys.argv[1:] or ["c1", "c2", "c3", "c4"]:
    dg = pg.make_config(name)
    torch.cuda.synchronize()
    pg.estimate_diameter(dg, samples=64, seed=0)      # warm-up
    t0 = time.perf_counter()
    s = pg.estimate_diameter(dg, samples=1000, seed=0)
    dt = time.perf_counter() - t0
    print(f"{name} n={s.n} m={s.m} diameter>={s.diameter_lower_bound} samples=1000 {dt:.3f}s", flush=True)
