"""Run one config + a few FAST-BCC calls (the target for ncu / compute-sanitizer).

    python tools/profile_run.py --config c5a --calls 2
    python tools/profile_run.py --rmat 26            # RMAT scale 26, avg degree 16
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2404_17101_b200 as pg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5a")
    ap.add_argument("--rmat", type=int, default=0, help="RMAT scale (avg degree 16) instead of --config")
    ap.add_argument("--calls", type=int, default=2)
    ap.add_argument("--canonical", action="store_true")
    a = ap.parse_args()
    if a.rmat:
        dg = pg.gen_rmat(a.rmat, 8 << a.rmat, seed=1)
    else:
        dg = pg.make_config(a.config)
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    r = None
    for _ in range(a.calls):
        r = pg.bcc_device(dg.offsets, dg.targets, canonical=a.canonical)
    torch.cuda.synchronize()
    print("n", dg.n, "M", dg.m, "bcc_count", int(r.bcc_count.item()), "launches/call", r.launches)


if __name__ == "__main__":
    main()
