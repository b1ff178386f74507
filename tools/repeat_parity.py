"""Race hunting: many BCC calls on one device graph with different sampling seeds and
canonical output; every call must give the same canonical labels, articulation bitmap
and count (the union-find schedule, and so the forest, changes from call to call).

    python tools/repeat_parity.py --config c4 --calls 20
"""
import argparse
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2404_17101_b200 as pg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--calls", type=int, default=20)
    a = ap.parse_args()
    dg = pg.make_config(a.config)
    ref = None
    for i in range(a.calls):
        r = pg.bcc_device(dg.offsets, dg.targets, seed=1000 + i, canonical=True, validate=(i == 0))
        torch.cuda.synchronize()
        hl = hashlib.blake2b(r.edge_label.cpu().numpy().view(np.uint8), digest_size=16).hexdigest()
        ha = hashlib.blake2b(r.artic_bits.cpu().numpy().view(np.uint8), digest_size=16).hexdigest()
        key = (hl, ha, int(r.bcc_count.item()))
        if ref is None:
            ref = key
        print(a.config, i, "ok" if key == ref else f"MISMATCH {key} vs {ref}", flush=True)
        if key != ref:
            return 1
    return 0


if __name__ == "__main__":
    sys.exit(main())
