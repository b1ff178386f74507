"""Pin the C oracle to the REAL reference at full BASELINE size (C2, C3, C4).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_fullsize_hashes.py [c2 c3 c4]

Runs pasgal.oracles.bcc_hopcroft_tarjan (oracles.py:119-201) -- the reference's own
Python code, unmodified -- on the full-size C2 (RMAT 2^20, 2^24 draws), C3 (grid 4096^2,
p=0.6) and C4 (kNN k=5, 2^25 points) CSRs built by this repo's host generator twins
(oracle/gen_host.c, whose outputs equal the device generators'), and commits only hashes:

* ``raw``: blake2b-128 of the reference's raw int64 ``_edge_label`` (its comp_count
  numbering, self-loop slots -1) -- the C oracle must reproduce it bit for bit
  (tests/test_oracle.py::test_oracle_full_size_vs_reference_hashes);
* ``labels``: blake2b-128 of the min-edge-id canonical labels derived from those raw labels
  with numpy here (uint32, 0xFFFFFFFF for unlabelled slots) -- what the device returns in
  PASGAL_BCC_CANONICAL mode (tests/test_gpu_parity.py compares against it directly);
* ``artic``: blake2b-128 of the reference's bool articulation array; ``count``, ``artic_count``.

/root/reference does not exist on the GPU box, so the hashes are committed
(tests/golden/fullsize_ref_hashes.json). Measured run times are recorded alongside.
"""

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

from pasgal.graph import Graph  # noqa: E402
from pasgal.oracles import bcc_hopcroft_tarjan  # noqa: E402

import oracle  # noqa: E402  (host generator twins only)

OUT = os.path.join(HERE, "fullsize_ref_hashes.json")


def h(a):
    return hashlib.blake2b(np.ascontiguousarray(a).view(np.uint8), digest_size=16).hexdigest()


def min_eid_labels(offsets, targets, raw):
    """Canonical labels (oracle_canonical_min_eid's definition, results.py:103-112 order):
    the undirected edge id of slot u->w with u < w is its rank among all such slots in CSR
    order; every slot gets the minimum id over its BCC; unlabelled slots 0xFFFFFFFF."""
    raw = np.asarray(raw, dtype=np.int64)
    m = raw.shape[0]
    n = offsets.shape[0] - 1
    src = np.repeat(np.arange(n, dtype=np.int64), np.diff(offsets))
    up = targets.astype(np.int64) > src
    del src
    eid = np.cumsum(up, dtype=np.int64) - 1
    out = np.full(m, 0xFFFFFFFF, dtype=np.uint32)
    ok = raw >= 0
    if ok.any():
        k = int(raw[ok].max()) + 1
        best = np.full(k, np.iinfo(np.int64).max, dtype=np.int64)
        sel = ok & up
        np.minimum.at(best, raw[sel], eid[sel])
        out[ok] = best[raw[ok]].astype(np.uint32)
    return out


def build(name):
    if name == "c2":
        return oracle.rmat(20, 1 << 24, seed=1)
    if name == "c3":
        return oracle.gen_grid(4096, 4096, 0.6, 1)
    if name == "c4":
        return oracle.knn(1 << 25, 5, seed=1)
    raise ValueError(name)


def main(names):
    res = json.load(open(OUT)) if os.path.exists(OUT) else {}
    res["_source"] = ("pasgal.oracles.bcc_hopcroft_tarjan (the unmodified Python reference) on the "
                      "host-twin CSRs of BASELINE configs[1..3]; tests/golden/make_fullsize_hashes.py")
    for name in names:
        off, tgt = build(name)
        t0 = time.time()
        r = bcc_hopcroft_tarjan(Graph(off, tgt))
        dt = time.time() - t0
        raw = np.asarray(r._edge_label, dtype=np.int64)
        art = np.asarray(r.articulation, dtype=bool)
        res[name] = dict(
            n=int(off.shape[0] - 1), m_slots=int(tgt.shape[0]),
            csr=h(off) + ":" + h(tgt),
            raw=h(raw), labels=h(min_eid_labels(off, tgt, raw)), artic=h(art),
            count=int(r.bcc_count), artic_count=int(art.sum()), reference_s=round(dt, 1))
        print(name, res[name], flush=True)
        with open(OUT, "w") as f:
            json.dump(res, f, indent=1, sort_keys=True)
        del r, raw, art, off, tgt


if __name__ == "__main__":
    main(sys.argv[1:] or ["c2", "c3", "c4"])
