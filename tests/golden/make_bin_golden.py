"""Generate tests/golden/bin_cases.json from the REAL reference's binary loader.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_bin_golden.py

Each case is a (file name, byte string) pair fed to the reference's own
``pasgal.graph.load_graph`` (graph.py:411-418, which dispatches to load_bin, graph.py:341-395,
or load_adj); the fixture records what it returned (n, m, offsets, targets) or the exception
type and message it raised, with the file path replaced by ``{path}``.  It covers the
``.wbin`` weight block (negative weight at edge i, NaN and -0.0 accepted), the extension
dispatch, and unknown extensions.  The device loader (paper_2404_17101_b200.io.load_graph)
must reproduce every case.  /root/reference does not exist on the GPU box, so the fixtures
are committed.
"""

import base64
import json
import os
import struct
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from pasgal.graph import load_graph  # noqa: E402


def binf(n, offsets, targets, weights=None, size=None, m=None):
    m = len(targets) if m is None else m
    size = 24 + (n + 1) * 8 + m * 4 if size is None else size
    b = struct.pack("<QQQ", n, m, size) + np.asarray(offsets, "<u8").tobytes() + np.asarray(targets, "<u4").tobytes()
    if weights is not None:
        b += np.asarray(weights, "<f4").tobytes()
    return b


def cases():
    tri_o, tri_t = [0, 2, 4, 6], [1, 2, 0, 2, 0, 1]
    c = [
        ("ok.bin", binf(3, tri_o, tri_t)),
        ("ok.wbin", binf(3, tri_o, tri_t, [1, 2, 3, 1, 2, 3])),
        ("ok_zero_weights.wbin", binf(3, tri_o, tri_t, [0, 0, 0, 0, 0, 0])),
        ("neg_first.wbin", binf(3, tri_o, tri_t, [-1, 2, 3, 1, 2, 3])),
        ("neg_mid.wbin", binf(3, tri_o, tri_t, [1, 2, 3, -0.5, -2, 3])),
        ("neg_last.wbin", binf(3, tri_o, tri_t, [1, 2, 3, 1, 2, -1e-30])),
        ("neg_inf.wbin", binf(3, tri_o, tri_t, [1, 2, float("-inf"), 1, 2, 3])),
        ("nan_weight.wbin", binf(3, tri_o, tri_t, [1, float("nan"), 3, 1, 2, 3])),
        ("negzero_weight.wbin", binf(3, tri_o, tri_t, [1, -0.0, 3, 1, 2, 3])),
        ("nan_then_neg.wbin", binf(3, tri_o, tri_t, [float("nan"), 1, 3, -4, 2, 3])),
        ("truncated_weights.wbin", binf(3, tri_o, tri_t, [1, 2, 3])),
        ("empty_graph.wbin", binf(2, [0, 0, 0], [], [])),
        ("bad_target.wbin", binf(3, tri_o, [1, 2, 0, 9, 0, 1], [-1, 2, 3, 1, 2, 3])),
        ("weights_ignored.bin", binf(3, tri_o, tri_t, [-1, -1, -1, -1, -1, -1])),
        ("unknown.txt", binf(3, tri_o, tri_t)),
        ("noext", binf(3, tri_o, tri_t)),
        ("upper.BIN", binf(3, tri_o, tri_t)),
        ("ok.adj", b"AdjacencyGraph\n3\n6\n0\n2\n4\n1\n2\n0\n2\n0\n1\n"),
    ]
    # a longer block: first negative weight deep inside
    n = 1000
    offs = np.arange(n + 1, dtype=np.int64)
    tg = (np.arange(n) + 1) % n
    w = np.ones(n, dtype=np.float32)
    w[777] = -3
    w[900] = -1
    c.append(("long_neg.wbin", binf(n, offs, tg, w)))
    return c


def main():
    out = []
    with tempfile.TemporaryDirectory() as d:
        for name, data in cases():
            p = os.path.join(d, name)
            with open(p, "wb") as f:
                f.write(data)
            rec = {"name": name, "data_b64": base64.b64encode(data).decode()}
            try:
                g = load_graph(p)
                rec["expect"] = {"n": int(g.n), "m": int(g.m), "offsets": g.offsets.tolist(),
                                 "targets": [int(t) for t in g.targets]}
            except Exception as e:  # noqa: BLE001
                rec["expect"] = {"error": type(e).__name__, "message": str(e).replace(p, "{path}")}
            out.append(rec)
    with open(os.path.join(HERE, "bin_cases.json"), "w") as f:
        json.dump(out, f, indent=0)
    for r in out:
        print(r["name"], r["expect"].get("error", "ok"), r["expect"].get("message", ""))


if __name__ == "__main__":
    main()
