"""One-off full-size parity: FAST-BCC on the device vs the C oracle on the host, for a
BASELINE config (default C5a, RMAT 2^28).  Device outputs are hashed then freed so the
oracle fits in host RAM; the canonical labels, articulation bitmap and bcc_count must
match exactly.  Writes a JSON summary (profiles/ keeps the round's result).

    python tools/full_parity.py --config c5a --out gpurun_out/c5a_parity.json
    python tools/full_parity.py --against profiles/r01_c5a_parity.json --seeds 0,7   # device only
"""
import argparse
import hashlib
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2404_17101_b200 as pg  # noqa: E402


def h(a):
    return hashlib.blake2b(np.ascontiguousarray(a).view(np.uint8), digest_size=16).hexdigest()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5a")
    ap.add_argument("--out", default="gpurun_out/full_parity.json")
    ap.add_argument("--against", default="",
                    help="device run only, compared with the oracle hashes of an earlier full run "
                         "(e.g. profiles/r01_c5a_parity.json)")
    ap.add_argument("--seeds", default="0", help="comma-separated BCC sampling seeds (device side)")
    a = ap.parse_args()
    t0 = time.time()
    dg = pg.make_config(a.config)
    n, m = dg.n, dg.m
    devs = []
    for seed in [int(x) for x in a.seeds.split(",")]:
        r = pg.bcc_device(dg.offsets, dg.targets, seed=seed, canonical=True, validate=True)
        torch.cuda.synchronize()
        lab = r.edge_label.cpu().numpy().view(np.uint32)
        art = pg.unpack_articulation(r.artic_bits.cpu().numpy(), n)
        cnt = int(r.bcc_count.item())
        devs.append({"seed": seed, "labels": h(lab), "artic": h(art), "count": cnt, "artic_count": int(art.sum())})
        del lab, art, r
    dev = devs[0]
    if a.against:
        with open(a.against) as f:
            refd = json.load(f)["oracle"]
        res = {"config": a.config, "n": n, "m_slots": m, "device": devs, "oracle": refd,
               "oracle_source": a.against, "total_seconds": round(time.time() - t0, 1),
               "match": all(d["labels"] == refd["labels"] and d["artic"] == refd["artic"] and
                            d["count"] == refd["count"] for d in devs)}
        os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)
        print(json.dumps(res))
        return 0 if res["match"] else 1
    off = dg.offsets.cpu().numpy()
    tgt = dg.targets.cpu().numpy().view(np.uint32)
    del dg
    pg.release_workspace()
    torch.cuda.empty_cache()
    t1 = time.time()
    ref = oracle.bcc_hopcroft_tarjan(off, tgt)
    t2 = time.time()
    ref_art = ref.articulation
    refd = {"artic": h(ref_art), "count": ref.bcc_count, "artic_count": int(ref_art.sum())}
    del ref_art
    want = oracle.canonical_min_eid(off, tgt, ref.edge_label)
    del ref
    refd["labels"] = h(want)
    res = {"config": a.config, "n": n, "m_slots": m, "device": dev, "oracle": refd,
           "oracle_seconds": round(t2 - t1, 1), "total_seconds": round(time.time() - t0, 1),
           "match": dev["labels"] == refd["labels"] and dev["artic"] == refd["artic"] and dev["count"] == refd["count"]}
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res))
    return 0 if res["match"] else 1


if __name__ == "__main__":
    sys.exit(main())
