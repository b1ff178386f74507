"""Device ms per FAST-BCC call for BASELINE configs (bench.py's time_device: fixed buffers,
L2 flushed between steps), optionally with env overrides, e.g.

    python tools/config_times.py c1 c2 c3 c4
    PASGAL_BCC_LOCAL_LB=11 python tools/config_times.py c1
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2404_17101_b200 as pg  # noqa: E402


def main():
    names = [a for a in sys.argv[1:] if not a.startswith("-")] or ["c1", "c2", "c3", "c4"]
    steps = 10
    res = {}
    for name in names:
        dg = pg.make_config(name)
        torch.cuda.synchronize()
        ms, nl = bench.time_device(pg, torch, dg, steps=steps, warmup=3)
        res[name] = {"ms": round(ms, 4), "launches": nl}
        if "--nograph" in sys.argv or name in ("c1", "c2"):
            bmod = sys.modules["paper_2404_17101_b200.bcc"]
            saved = bmod.GRAPH_MAX_N
            bmod.GRAPH_MAX_N = 0
            ms2, _ = bench.time_device(pg, torch, dg, steps=steps, warmup=3)
            bmod.GRAPH_MAX_N = saved
            res[name]["ms_no_graph"] = round(ms2, 4)
        del dg
        pg.release_workspace()
        torch.cuda.empty_cache()
    print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("PASGAL")}, "configs": res}))


if __name__ == "__main__":
    main()
