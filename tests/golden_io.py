"""Loader for the committed golden fixtures (tests/golden/*.npz, made by make_golden.py
from the real reference)."""

import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


class Case:
    def __init__(self, offsets, targets, label, artic, count, canon, name=""):
        self.offsets = np.asarray(offsets, dtype=np.int64)
        self.targets = np.asarray(targets, dtype=np.uint32)
        self.label = np.asarray(label, dtype=np.int32)
        n = self.offsets.shape[0] - 1
        self.articulation = np.unpackbits(np.asarray(artic, dtype=np.uint8), bitorder="little")[:n].astype(bool)
        self.count = int(count)
        self.canon = np.asarray(canon, dtype=np.int64)
        self.name = name

    @property
    def n(self):
        return self.offsets.shape[0] - 1

    @property
    def m(self):
        return self.targets.shape[0]


def _unpack(z, names=None):
    keys = ["offsets", "targets", "label", "artic", "canon"]
    k = z["count"].shape[0]
    out = []
    for i in range(k):
        parts = {}
        for key in keys:
            a, b = z[key + "_idx"][i], z[key + "_idx"][i + 1]
            parts[key] = z[key][a:b]
        out.append(Case(parts["offsets"], parts["targets"], parts["label"], parts["artic"], z["count"][i],
                        parts["canon"], names[i] if names is not None else f"corpus{i}"))
    return out


def kats():
    z = np.load(os.path.join(GOLDEN, "kats.npz"))
    return _unpack(z, [str(s) for s in z["names"]])


def corpus():
    return _unpack(np.load(os.path.join(GOLDEN, "corpus.npz")))


def single(fname):
    z = np.load(os.path.join(GOLDEN, fname))
    return Case(z["offsets"], z["targets"], z["label"], z["artic"], z["count"], z["canon"], fname)


SINGLES = ["c1_grid256_p06_s1.npz", "rmat_s12_d16_seed7.npz", "knn_13_k5_seed3.npz"]


def all_cases():
    return kats() + corpus() + [single(f) for f in SINGLES]


def dense_from_min_eid(case, canon_u32):
    """canonical_edge_partition-equivalent dense ids from per-slot min-eid labels."""
    src = np.repeat(np.arange(case.n, dtype=np.int64), np.diff(case.offsets))
    up = src < case.targets.astype(np.int64)
    _, dense = np.unique(np.asarray(canon_u32)[up].astype(np.int64), return_inverse=True)
    return dense.reshape(-1)
