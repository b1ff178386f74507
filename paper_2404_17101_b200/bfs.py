"""Device BFS and sampled diameter estimation.

``bfs`` returns the exact hop distances of the reference's ``oracles.bfs_queue``
(oracles.py:27-46) as a ``DistanceArray`` (results.py:9-19); ``estimate_diameter`` is the
reference's ``estimate_diameter`` (graph.py:595-605): the same ``default_rng(seed)`` source
sample, the same max-eccentricity bound, returned as ``GraphStats`` (graph.py:130-137).
Both run the bit-parallel multi-source BFS of csrc/bfs.cu: up to 64 sampled sources share
one traversal, so 1000 samples cost at most 16 device BFS passes.

On an undirected (symmetric) graph the estimate also bounds before it searches: each pass
records the hop distance from its sources to every other sampled source, and since
ecc(x) <= d(x, s) + ecc(s), a sample whose bound is already <= the best eccentricity found
cannot change the maximum and is never run.  Samples run highest-bound first.  The result
is exactly the reference's max over all samples; directed graphs run every sample.
"""

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .graph import DeviceGraph

UNREACHED = -1
_MAX_SOURCES = 64


class DistanceArray:
    """Exact hop distances from a source; UNREACHED (-1) where unreachable."""

    __slots__ = ("dist", "source", "rounds")

    def __init__(self, dist, source, rounds=0):
        self.dist = np.asarray(dist, dtype=np.int64)
        self.source = int(source)
        self.rounds = int(rounds)


@dataclass
class GraphStats:
    """Sampled eccentricity statistics; the bound never exceeds the diameter."""

    n: int
    m: int
    diameter_lower_bound: int
    sample_count: int


def _device_csr(g, device):
    if isinstance(g, DeviceGraph):
        return g.offsets, g.targets
    off = torch.from_numpy(np.ascontiguousarray(g.offsets, dtype=np.int64)).to(device)
    tgt = np.asarray(g.targets)
    if tgt.shape[0] and (int(tgt.max()) >= off.shape[0] - 1 or int(tgt.min()) < 0):
        raise ValueError("edge target out of range")
    tgt = torch.from_numpy(np.ascontiguousarray(tgt.astype(np.int32, copy=False).view(np.int32))).to(device)
    return off, tgt


class _Msbfs:
    def __init__(self, off, tgt):
        self.lib = _lib.load()
        self.off, self.tgt = off, tgt
        self.n = off.shape[0] - 1
        self.ws = torch.empty(int(self.lib.pasgal_msbfs_workspace_bytes(self.n)), dtype=torch.uint8,
                              device=off.device)
        self.csr = _lib.PasgalCsr(self.n, tgt.shape[0], off.data_ptr(), tgt.data_ptr() if tgt.shape[0] else 0)
        self.stream = ctypes.c_void_p(torch.cuda.current_stream(off.device).cuda_stream)

    def run(self, sources, dist=None, probe=None, probe_dist=None):
        k = len(sources)
        src = (ctypes.c_int64 * k)(*[int(s) for s in sources])
        ecc = (ctypes.c_int64 * k)()
        levels = ctypes.c_int64()
        nprobe = 0 if probe_dist is None else probe_dist.shape[1]
        vp = lambda t: ctypes.c_void_p(t.data_ptr() if t is not None else 0)  # noqa: E731
        st = self.lib.pasgal_msbfs_ex(ctypes.byref(self.csr), src, k, vp(dist), ecc, ctypes.byref(levels),
                                      vp(probe), nprobe, vp(probe_dist), vp(self.ws), self.ws.numel(), self.stream)
        _lib.check(st, "msbfs")
        return [int(e) for e in ecc], int(levels.value)


def bfs(g, source, device="cuda"):
    """Exact hop distances from ``source`` (oracles.bfs_queue, oracles.py:27-46)."""
    off, tgt = _device_csr(g, device)
    n = off.shape[0] - 1
    if not 0 <= source < n:
        raise ValueError(f"source {source} out of range for n={n}")
    dist = torch.empty(n, dtype=torch.int32, device=off.device)
    _, levels = _Msbfs(off, tgt).run([source], dist)
    return DistanceArray(dist.cpu().numpy().astype(np.int64), source, rounds=levels)


@dataclass
class VgcConfig:
    """SPEC.md vgc-engine VgcConfig: ``tau`` = minimum vertices a local search processes
    (>= 1), ``max_local_queue`` = its working-set cap (>= tau; the device queue holds 256
    vertices per warp and overflows to the next frontier), ``dense_threshold`` = fraction of
    m above which a round runs bottom-up (symmetric graphs; the spec's 0 < t < 1, with 0 =
    always and 1 = never allowed for the self-equivalence tests)."""

    tau: int = 512
    max_local_queue: int = 2048
    dense_threshold: float = 1 / 20

    def __post_init__(self):
        if not (1 <= self.tau <= self.max_local_queue):
            raise ValueError("need 1 <= tau <= max_local_queue")
        if not 0 <= self.dense_threshold <= 1:
            raise ValueError("need 0 <= dense_threshold <= 1")


def bfs_parallel(g, source, cfg=None, device="cuda", symmetric=None, return_stats=False):
    """SPEC.md bfs_parallel: exact hop distances from ``source`` by the VGC frontier engine
    (csrc/vgc.cu; pasgal_bfs_vgc_ex): rounds of per-warp multi-hop local searches with
    write-min distances, and on a symmetric graph dense (bottom-up) rounds when the
    frontier's out-degree sum exceeds ``cfg.dense_threshold * m`` (bfs_round_dense).
    ``symmetric``: None checks it on the device (only when dense rounds can trigger).
    Returns a DistanceArray whose ``rounds`` is the number of frontier rounds (tau = 1 and no
    dense rounds: level-synchronous, eccentricity + 1 rounds); with ``return_stats`` also
    ``{"dense_rounds": k}``."""
    cfg = cfg or VgcConfig()
    off, tgt = _device_csr(g, device)
    n = off.shape[0] - 1
    if not 0 <= source < n:
        raise ValueError(f"source {source} out of range for n={n}")
    if symmetric is None:
        symmetric = cfg.dense_threshold < 1 and _is_symmetric(off, tgt)
    lib = _lib.load()
    dist = torch.empty(n, dtype=torch.int32, device=off.device)
    ws = torch.empty(int(lib.pasgal_bfs_vgc_workspace_bytes(n)), dtype=torch.uint8, device=off.device)
    csr = _lib.PasgalCsr(n, tgt.shape[0], off.data_ptr(), tgt.data_ptr() if tgt.shape[0] else 0)
    rounds, dense = ctypes.c_int64(), ctypes.c_int64()
    st = lib.pasgal_bfs_vgc_ex(ctypes.byref(csr), int(source), int(cfg.tau), float(cfg.dense_threshold),
                               int(bool(symmetric)), ctypes.c_void_p(dist.data_ptr()), ctypes.byref(rounds),
                               ctypes.byref(dense), ctypes.c_void_p(ws.data_ptr()), ws.numel(),
                               ctypes.c_void_p(torch.cuda.current_stream(off.device).cuda_stream))
    _lib.check(st, "bfs_vgc")
    res = DistanceArray(dist.cpu().numpy().astype(np.int64), source, rounds=int(rounds.value))
    return (res, {"dense_rounds": int(dense.value)}) if return_stats else res


def eccentricities(g, sources, device="cuda"):
    """Eccentricity (max hop distance reached) of every source, 64 per device pass."""
    off, tgt = _device_csr(g, device)
    eng = _Msbfs(off, tgt)
    out = []
    for i in range(0, len(sources), _MAX_SOURCES):
        out += eng.run(sources[i:i + _MAX_SOURCES])[0]
    return out


def _is_symmetric(off, tgt):
    from .bcc import validate_device

    try:
        validate_device(off, tgt)
        return True
    except ValueError:           # not symmetric (or unsorted rows): no bounding
        return False


def _bounded_max_ecc(off, tgt, uniq):
    """max ecc over `uniq` on a symmetric graph, skipping samples bounded by the best."""
    eng = _Msbfs(off, tgt)
    k = len(uniq)
    probe = torch.full((eng.n,), -1, dtype=torch.int32, device=off.device)
    probe[torch.tensor(uniq, dtype=torch.int64, device=off.device)] = torch.arange(k, dtype=torch.int32,
                                                                                 device=off.device)
    pd = torch.empty((_MAX_SOURCES, k), dtype=torch.int32, device=off.device)
    ub = np.full(k, np.iinfo(np.int64).max, dtype=np.int64)
    todo = np.ones(k, dtype=bool)
    best = -1
    passes = 0
    while todo.any():
        cand = np.flatnonzero(todo)
        batch = cand[np.argsort(-ub[cand], kind="stable")][:_MAX_SOURCES]
        ecc, _ = eng.run([uniq[j] for j in batch], probe=probe, probe_dist=pd[:len(batch)])
        passes += 1
        todo[batch] = False
        best = max(best, max(ecc))
        d = pd[:len(batch)].cpu().numpy().astype(np.int64)        # d[i, j] = dist(batch[i], uniq[j])
        bound = np.where(d >= 0, d + np.asarray(ecc, np.int64)[:, None], np.iinfo(np.int64).max).min(axis=0)
        ub = np.minimum(ub, bound)
        todo &= ub > best
    return best, passes


def estimate_diameter(g, samples=1000, seed=0, device="cuda", bound=True):
    """Lower-bound the diameter by the max eccentricity of sampled sources
    (graph.py:595-605: same validation, same numpy source stream, same bound).  With
    ``bound`` (default) a symmetric graph skips samples that provably cannot raise it."""
    if samples < 1:
        raise ValueError("samples must be >= 1")
    off, tgt = _device_csr(g, device)
    n, m = off.shape[0] - 1, tgt.shape[0]
    if n == 0 or m == 0:
        return GraphStats(n, m, 0, samples)
    rng = np.random.default_rng(seed)
    sources = rng.integers(0, n, size=samples, dtype=np.int64)
    uniq = list(dict.fromkeys(sources.tolist()))
    if bound and len(uniq) > _MAX_SOURCES and _is_symmetric(off, tgt):
        best, _ = _bounded_max_ecc(off, tgt, uniq)
    else:
        best = max(eccentricities(DeviceGraph(off, tgt), uniq, device))
    return GraphStats(n, m, int(best), samples)
