"""oracle -- TEST INFRASTRUCTURE ONLY: the CPU parity checker.

This package is the checker, never the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import it.  ``paper_2404_17101_b200`` never does.

* ``bcc_hopcroft_tarjan`` -- plain-C restatement (bcc_oracle.c) of the reference's
  sequential oracle ``pasgal.oracles.bcc_hopcroft_tarjan``
  (/root/reference/pkg/src/pasgal/oracles.py:119-201), including its
  ``is_symmetric`` precondition (graph.py:123-158) and ``_twin_edges``
  (oracles.py:107-116).  Pinned against the reference itself through the golden
  fixtures in ``tests/golden/`` (made by ``tests/golden/make_golden.py``, which imports
  the reference in the build container): raw labels, articulation and bcc_count match
  the reference bit for bit, before any canonicalisation.
* ``canonical_min_eid`` -- the parity comparator: every slot labelled by the minimum
  undirected edge id of its BCC (order-isomorphic to
  ``results.canonical_edge_partition``, results.py:103-112).
* ``bfs_queue`` / ``estimate_diameter`` -- C restatement of the reference's FIFO BFS
  (oracles.py:27-46, graph.py:557-605), pinned by tests/golden/bfs_cases.npz.
* ``gen_grid`` / ``rmat`` / ``knn`` -- host twins of the device generators
  (rules pinned in DESIGN.md, "Generators").
"""

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

_i64p = ctypes.POINTER(ctypes.c_int64)
_u32p = ctypes.POINTER(ctypes.c_uint32)
_i32p = ctypes.POINTER(ctypes.c_int32)
_u8p = ctypes.POINTER(ctypes.c_uint8)
_u64p = ctypes.POINTER(ctypes.c_uint64)


def build():
    """Compile liboracle.so (gcc, seconds)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        build()
    lib = ctypes.CDLL(_LIB_PATH)
    lib.oracle_bcc_hopcroft_tarjan.argtypes = [ctypes.c_int64, _i64p, _u32p, _i32p, _u8p, _i64p]
    lib.oracle_bcc_hopcroft_tarjan.restype = ctypes.c_int
    lib.oracle_is_symmetric.argtypes = [ctypes.c_int64, _i64p, _u32p]
    lib.oracle_is_symmetric.restype = ctypes.c_int
    lib.oracle_canonical_min_eid.argtypes = [ctypes.c_int64, _i64p, _u32p, _i32p, ctypes.c_int64, _u32p]
    lib.oracle_canonical_min_eid.restype = ctypes.c_int
    lib.oracle_connected_components.argtypes = [ctypes.c_int64, _i64p, _u32p, _i32p]
    lib.oracle_connected_components.restype = ctypes.c_int64
    lib.oracle_bfs.argtypes = [ctypes.c_int64, _i64p, _u32p, ctypes.c_int64, _i32p]
    lib.oracle_bfs.restype = ctypes.c_int64
    lib.oracle_count_upper.argtypes = [ctypes.c_int64, _i64p, _u32p]
    lib.oracle_count_upper.restype = ctypes.c_int64
    lib.host_csr_from_keys.argtypes = [ctypes.c_int64, _u64p, ctypes.c_int64, _i64p, _u32p]
    lib.host_csr_from_keys.restype = ctypes.c_int64
    lib.host_gen_grid.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint64,
                                  ctypes.c_int, _i64p, _u32p]
    lib.host_gen_grid.restype = ctypes.c_int64
    lib.host_rmat_keys.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint32,
                                   ctypes.c_uint32, ctypes.c_uint32, _u64p]
    lib.host_rmat_keys.restype = ctypes.c_int64
    lib.host_knn_points.argtypes = [ctypes.c_int64, ctypes.c_uint64, _u32p, _u32p]
    lib.host_knn_points.restype = None
    lib.host_knn_keys.argtypes = [ctypes.c_int64, ctypes.c_int, _u32p, _u32p, ctypes.c_int, _u64p]
    lib.host_knn_keys.restype = ctypes.c_int64
    lib.host_knn_keys_brute.argtypes = [ctypes.c_int64, ctypes.c_int, _u32p, _u32p, _u64p]
    lib.host_knn_keys_brute.restype = ctypes.c_int64
    _lib = lib
    return lib


def _p(a, t):
    return a.ctypes.data_as(t)


def _csr(offsets, targets):
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    tgt = np.ascontiguousarray(targets, dtype=np.uint32)
    if off.shape[0] < 1 or off[-1] != tgt.shape[0]:
        raise ValueError("offsets[n] must equal len(targets)")
    return off, tgt


class OracleBcc:
    """Oracle output: same fields as the reference's BccLabels in edge-label mode."""

    __slots__ = ("edge_label", "articulation", "bcc_count")

    def __init__(self, edge_label, articulation, bcc_count):
        self.edge_label = edge_label
        self.articulation = articulation
        self.bcc_count = bcc_count


def bcc_hopcroft_tarjan(offsets, targets):
    """oracles.py:119-201 restated in C.  Raises ValueError on a non-symmetric graph."""
    lib = _load()
    off, tgt = _csr(offsets, targets)
    n = off.shape[0] - 1
    lab = np.empty(max(tgt.shape[0], 1), dtype=np.int32)
    art = np.empty(max(n, 1), dtype=np.uint8)
    cnt = np.zeros(1, dtype=np.int64)
    st = lib.oracle_bcc_hopcroft_tarjan(n, _p(off, _i64p), _p(tgt, _u32p), _p(lab, _i32p),
                                        _p(art, _u8p), _p(cnt, _i64p))
    if st == 2:
        raise ValueError("biconnectivity requires a symmetric graph")
    if st != 0:
        raise MemoryError("oracle allocation failed")
    return OracleBcc(lab[: tgt.shape[0]], art[:n].astype(bool), int(cnt[0]))


def is_symmetric(offsets, targets):
    lib = _load()
    off, tgt = _csr(offsets, targets)
    r = lib.oracle_is_symmetric(off.shape[0] - 1, _p(off, _i64p), _p(tgt, _u32p))
    if r < 0:
        raise MemoryError("oracle allocation failed")
    return bool(r)


def canonical_min_eid(offsets, targets, labels):
    """Per slot: the minimum undirected edge id (rank of the u<w slot in CSR order) of
    its class.  Rows must be sorted.  Returns uint32[M]."""
    lib = _load()
    off, tgt = _csr(offsets, targets)
    lab = np.ascontiguousarray(labels)
    if lab.dtype != np.int32:
        # arbitrary ids (e.g. device comp ids): densify first
        _, lab = np.unique(lab, return_inverse=True)
        lab = lab.astype(np.int32)
    nl = int(lab.max()) + 1 if lab.shape[0] else 0
    out = np.empty(max(tgt.shape[0], 1), dtype=np.uint32)
    st = lib.oracle_canonical_min_eid(off.shape[0] - 1, _p(off, _i64p), _p(tgt, _u32p),
                                      _p(lab, _i32p), nl, _p(out, _u32p))
    if st != 0:
        raise MemoryError("oracle allocation failed")
    return out[: tgt.shape[0]]


def connected_components(offsets, targets):
    """Components labelled by their minimum vertex id (BFS in increasing start order);
    restates SPEC.md:413-420 (the reference ships no code for it).  Returns (int32[n], count)."""
    lib = _load()
    off, tgt = _csr(offsets, targets)
    n = off.shape[0] - 1
    comp = np.empty(max(n, 1), dtype=np.int32)
    c = lib.oracle_connected_components(n, _p(off, _i64p), _p(tgt, _u32p), _p(comp, _i32p))
    if c < 0:
        raise MemoryError("oracle allocation failed")
    return comp[:n], int(c)


def bfs_queue(offsets, targets, source):
    """oracles.bfs_queue (oracles.py:27-46) in C: (dist int64[n] with -1 = unreachable,
    eccentricity of the source)."""
    lib = _load()
    off, tgt = _csr(offsets, targets)
    n = off.shape[0] - 1
    if not 0 <= source < n:
        raise ValueError(f"source {source} out of range for n={n}")
    dist = np.empty(max(n, 1), dtype=np.int32)
    ecc = lib.oracle_bfs(n, _p(off, _i64p), _p(tgt, _u32p), int(source), _p(dist, _i32p))
    if ecc < 0:
        raise MemoryError("oracle allocation failed")
    return dist[:n].astype(np.int64), int(ecc)


def estimate_diameter(offsets, targets, samples=1000, seed=0):
    """graph.estimate_diameter (graph.py:595-605): max eccentricity over the reference's
    default_rng(seed) source sample, one C BFS per source."""
    off, tgt = _csr(offsets, targets)
    n, m = off.shape[0] - 1, tgt.shape[0]
    if samples < 1:
        raise ValueError("samples must be >= 1")
    if n == 0 or m == 0:
        return 0
    sources = np.random.default_rng(seed).integers(0, n, size=samples, dtype=np.int64)
    return max(bfs_queue(off, tgt, int(s))[1] for s in sources)


def count_upper(offsets, targets):
    lib = _load()
    off, tgt = _csr(offsets, targets)
    return int(lib.oracle_count_upper(off.shape[0] - 1, _p(off, _i64p), _p(tgt, _u32p)))


# --------------------------------------------------------------------------------------
# generator twins (rules: DESIGN.md "Generators")
# --------------------------------------------------------------------------------------

def grid_threshold(p):
    """keep iff draw < floor(p * 2^64); p >= 1 keeps every lattice edge."""
    if p >= 1.0:
        return 0, 1
    return int(float(p) * 2.0 ** 64), 0


def rmat_thresholds(a, b, c):
    s = 2.0 ** 32
    return (min(int(a * s), 2 ** 32 - 1), min(int((a + b) * s), 2 ** 32 - 1),
            min(int((a + b + c) * s), 2 ** 32 - 1))


def gen_grid(rows, cols, p=0.6, seed=1):
    lib = _load()
    thr, keep_all = grid_threshold(p)
    n = rows * cols
    off = np.empty(n + 1, dtype=np.int64)
    tgt = np.empty(max(4 * n, 1), dtype=np.uint32)
    M = lib.host_gen_grid(rows, cols, seed, thr, keep_all, _p(off, _i64p), _p(tgt, _u32p))
    return off, tgt[:M].copy()


def csr_from_keys(n, keys):
    lib = _load()
    keys = np.ascontiguousarray(keys, dtype=np.uint64).copy()
    off = np.empty(n + 1, dtype=np.int64)
    tgt = np.empty(max(keys.shape[0], 1), dtype=np.uint32)
    M = lib.host_csr_from_keys(n, _p(keys, _u64p), keys.shape[0], _p(off, _i64p), _p(tgt, _u32p))
    if M < 0:
        raise MemoryError("oracle allocation failed")
    return off, tgt[:M].copy()


def rmat(scale, draws, seed=1, a=0.57, b=0.19, c=0.19):
    lib = _load()
    ta, tab, tabc = rmat_thresholds(a, b, c)
    keys = np.empty(max(2 * draws, 1), dtype=np.uint64)
    k = lib.host_rmat_keys(scale, draws, seed, ta, tab, tabc, _p(keys, _u64p))
    return csr_from_keys(1 << scale, keys[:k])


def knn_points(npts, seed=1):
    lib = _load()
    X = np.empty(max(npts, 1), dtype=np.uint32)
    Y = np.empty(max(npts, 1), dtype=np.uint32)
    lib.host_knn_points(npts, seed, _p(X, _u32p), _p(Y, _u32p))
    return X[:npts], Y[:npts]


def knn_gbits(npts):
    """Cell grid G = 2^g with G^2 <= npts/2 (about two points per cell), g in [0, 12]."""
    g = 0
    while g < 12 and (1 << (2 * (g + 1))) <= max(npts // 2, 1):
        g += 1
    return g


def knn(npts, k=5, seed=1, brute=False):
    lib = _load()
    if not 1 <= k <= 64:
        raise ValueError("k must be in [1, 64]")
    X, Y = knn_points(npts, seed)
    keys = np.empty(max(2 * k * npts, 1), dtype=np.uint64)
    if brute:
        nk = lib.host_knn_keys_brute(npts, k, _p(X, _u32p), _p(Y, _u32p), _p(keys, _u64p))
    else:
        nk = lib.host_knn_keys(npts, k, _p(X, _u32p), _p(Y, _u32p), knn_gbits(npts), _p(keys, _u64p))
    if nk < 0:
        raise MemoryError("oracle allocation failed")
    return csr_from_keys(npts, keys[:nk])
