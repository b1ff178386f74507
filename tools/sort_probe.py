"""CSR builder timing (RMAT keys -> sorted, deduplicated CSR) and equality of the onesweep
and legacy sorts: python tools/sort_probe.py SCALE"""
import hashlib
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2404_17101_b200 as pg  # noqa: E402


def run(scale):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dg = pg.gen_rmat(scale, 8 << scale, seed=1)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    h = hashlib.blake2b(dg.offsets.cpu().numpy().tobytes(), digest_size=8).hexdigest()
    h += ":" + hashlib.blake2b(dg.targets[: min(dg.m, 1 << 28)].cpu().numpy().tobytes(), digest_size=8).hexdigest()
    m = dg.m
    del dg
    torch.cuda.empty_cache()
    return dt, h, m


scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
run(min(scale, 20))                     # warm-up (module load, attributes)
dt, h, m = run(scale)
print(json.dumps({"scale": scale, "m_slots": m, "gen_s": round(dt, 4), "hash": h,
                  "legacy": bool(os.environ.get("PASGAL_SORT_LEGACY"))}))
