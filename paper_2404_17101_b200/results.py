"""Output container and parity comparator, mirroring the reference's results module.

* ``BccLabels`` -- same interface as pasgal.results.BccLabels (results.py:45-88):
  ``articulation`` (bool[n]), ``bcc_count``, ``articulation_count`` and
  ``edge_labels(g)``.  Both storage modes are supported: per-slot labels (what the device
  pipeline returns) and the parallel mode's comp/parent/first from which labels derive by
  the FAST-BCC rule (results.py:76-88: a tree edge takes its child's component, any other
  edge the component of the endpoint with the larger preorder rank).
* ``canonical_relabel`` / ``canonical_edge_partition`` -- the reference's comparator
  (results.py:91-112): undirected (u<v) slots in key order, renumbered by first occurrence.

These are host-side data-structure helpers (numpy), not the compute path.
"""

import numpy as np

UNLABELLED = np.uint32(0xFFFFFFFF)


def _slot_sources(offsets):
    offsets = np.asarray(offsets, dtype=np.int64)
    return np.repeat(np.arange(offsets.shape[0] - 1, dtype=np.int64), np.diff(offsets))


class BccLabels:
    """Per-edge biconnected-component ids plus articulation flags (results.py:45-88)."""

    __slots__ = ("articulation", "bcc_count", "_edge_label", "_comp", "_parent", "_first")

    def __init__(self, articulation, bcc_count, edge_label=None, comp=None, parent=None, first=None):
        self.articulation = np.asarray(articulation, dtype=bool)
        self.bcc_count = int(bcc_count)
        self._edge_label = edge_label
        self._comp = comp
        self._parent = parent
        self._first = first
        if edge_label is None and (comp is None or parent is None or first is None):
            raise ValueError("need either edge labels or comp+parent+first")

    @property
    def articulation_count(self):
        return int(np.count_nonzero(self.articulation))

    @property
    def raw_edge_label(self):
        """Per-slot labels as produced by the device (uint32, 0xFFFFFFFF = unlabelled)."""
        return self._edge_label

    def edge_labels(self, g):
        """int64 label of every directed slot of ``g`` (both directions equal; -1 = none)."""
        if self._edge_label is not None:
            lab = np.asarray(self._edge_label)
            if lab.dtype == np.uint32:
                out = lab.astype(np.int64)
                out[lab == UNLABELLED] = -1
                return out
            return lab.astype(np.int64, copy=False)
        comp = np.asarray(self._comp, dtype=np.int64)
        first = np.asarray(self._first, dtype=np.int64)
        src = _slot_sources(g.offsets)
        dst = np.asarray(g.targets).astype(np.int64)
        # the larger-preorder endpoint is the child of a tree edge, the deeper end of a back
        # edge, and either end of a cross edge (both share one skeleton component)
        lab = np.where(first[src] > first[dst], comp[src], comp[dst])
        lab[src == dst] = -1
        return lab


def canonical_relabel(labels):
    """Renumber labels 0, 1, 2, ... in order of first occurrence."""
    labels = np.asarray(labels)
    if labels.shape[0] == 0:
        return labels.astype(np.int64)
    uniq, inv = np.unique(labels, return_inverse=True)
    inv = inv.reshape(-1)
    first_pos = np.full(uniq.shape[0], labels.shape[0], dtype=np.int64)
    np.minimum.at(first_pos, inv, np.arange(labels.shape[0], dtype=np.int64))
    rank = np.empty(uniq.shape[0], dtype=np.int64)
    rank[np.argsort(first_pos)] = np.arange(uniq.shape[0], dtype=np.int64)
    return rank[inv]


def canonical_edge_partition(g, bcc):
    """Canonical labels of the undirected (u<v) slots in (u, v) key order."""
    lab = bcc.edge_labels(g)
    src = _slot_sources(g.offsets)
    dst = np.asarray(g.targets).astype(np.int64)
    up = src < dst
    n = np.asarray(g.offsets).shape[0] - 1
    order = np.argsort(src[up] * max(n, 1) + dst[up], kind="stable")
    return canonical_relabel(lab[up][order])


def min_eid_to_partition(g, canon_labels):
    """Dense first-occurrence ids from per-slot min-edge-id labels (CANONICAL mode).

    For sorted rows the min undirected edge id of a BCC is the position of its first
    (u<v) slot, so the dense rank of the min id equals canonical_edge_partition."""
    src = _slot_sources(g.offsets)
    dst = np.asarray(g.targets).astype(np.int64)
    up = src < dst
    ids = np.asarray(canon_labels)[up].astype(np.int64)
    _, dense = np.unique(ids, return_inverse=True)
    return dense.reshape(-1).astype(np.int64)


_CHK_MUL = 0x9E3779B1


def canonical_checksum(canon_labels, articulation, bcc_count):
    """Order-independent run checksum: (bcc_count, number of
    articulation points, sum over slots of canon[s] * w(s) mod 2^64) with canon the
    min-undirected-edge-id labels (uint32, 0xFFFFFFFF for self-loops) and the odd weight
    w(s) = ((s * 0x9E3779B1) mod 2^32) | 1.  canonical_checksum_device is its device twin."""
    lab = np.asarray(canon_labels).view(np.uint32).astype(np.uint64)
    s = np.arange(lab.shape[0], dtype=np.uint64)
    w = ((s * np.uint64(_CHK_MUL)) & np.uint64(0xFFFFFFFF)) | np.uint64(1)
    h = int((lab * w).sum(dtype=np.uint64)) if lab.shape[0] else 0
    return int(bcc_count), int(np.count_nonzero(articulation)), h
