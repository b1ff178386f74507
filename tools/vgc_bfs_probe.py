"""VGC frontier engine vs the bit-parallel BFS: rounds and wall time per config/tau."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2404_17101_b200 as pg  # noqa: E402

out = {}
for name in sys.argv[1:] or ["c3", "c4", "c2"]:
    dg = pg.make_config(name)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ref = pg.bfs(dg, 0)
    t_ms = (time.perf_counter() - t0) * 1e3
    row = {"msbfs_ms": round(t_ms, 2), "levels": int(ref.dist.max()) + 1}
    for tau in (1, 64, 1024, 8192):
        pg.bfs_parallel(dg, 0, pg.VgcConfig(tau=tau, max_local_queue=max(tau, 2048)))   # warm
        t0 = time.perf_counter()
        r = pg.bfs_parallel(dg, 0, pg.VgcConfig(tau=tau, max_local_queue=max(tau, 2048)))
        dt = (time.perf_counter() - t0) * 1e3
        row[f"tau{tau}"] = {"ms": round(dt, 2), "rounds": r.rounds, "exact": bool(np.array_equal(r.dist, ref.dist))}
    out[name] = row
    del dg
    torch.cuda.empty_cache()
print(json.dumps(out))
