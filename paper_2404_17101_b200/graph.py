"""CSR graphs on the B200: container, device CSR builder and seeded generators.

Mirrors the parts of the reference's graph core on the BCC path (graph.py:54-129 Graph,
176-194 from_edges, 452-481 symmetrize, 488-508 gen_grid) and adds the generators the
BASELINE configs need (grid with edge-keep probability, RMAT, kNN), all running on the
device through libpasgal_bcc.so.  Generator rules are pinned in DESIGN.md "Generators".

Device CSR layout: offsets int64[n+1], targets int32[M], rows sorted,
symmetric, duplicate- and self-loop-free.
"""

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib


def _ptr(t):
    return ctypes_void(t.data_ptr()) if t is not None else None


def ctypes_void(p):
    import ctypes

    return ctypes.c_void_p(p)


def _stream(device=None):
    return ctypes_void(torch.cuda.current_stream(device).cuda_stream)


@dataclass
class DeviceGraph:
    """Symmetric CSR resident in HBM (the pasgal_csr_t of the C-ABI)."""

    offsets: torch.Tensor   # int64 [n+1], cuda
    targets: torch.Tensor   # int32 [M], cuda

    @property
    def n(self):
        return self.offsets.shape[0] - 1

    @property
    def m(self):
        return self.targets.shape[0]

    def to_host(self):
        return Graph(self.offsets.cpu().numpy(), self.targets.cpu().numpy().view(np.uint32))


class Graph:
    """Host CSR with the reference Graph's attributes (offsets int64[n+1], targets
    uint32[M]).  Any object with ``offsets``/``targets`` (e.g. a pasgal Graph) is accepted
    wherever a Graph is expected."""

    __slots__ = ("offsets", "targets")

    def __init__(self, offsets, targets):
        self.offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        t = np.ascontiguousarray(targets)
        if t.dtype == np.int32:
            t = t.view(np.uint32)
        elif t.dtype != np.uint32:
            t = t.astype(np.uint32)
        self.targets = t
        if self.offsets.shape[0] < 1 or int(self.offsets[-1]) != self.targets.shape[0]:
            raise ValueError(f"offsets[n]={int(self.offsets[-1]) if self.offsets.shape[0] else None} "
                             f"!= m={self.targets.shape[0]}")

    @property
    def n(self):
        return self.offsets.shape[0] - 1

    @property
    def m(self):
        return self.targets.shape[0]

    def to_device(self, device="cuda", pinned=False):
        off = torch.from_numpy(self.offsets)
        tgt = torch.from_numpy(self.targets.view(np.int32))
        if pinned:
            off, tgt = off.pin_memory(), tgt.pin_memory()
        return DeviceGraph(off.to(device, non_blocking=pinned), tgt.to(device, non_blocking=pinned))

    def __repr__(self):
        return f"Graph(n={self.n}, m={self.m})"


def _read_scalar(t):
    return int(t.item())


# ----------------------------------------------------------------------------------------
# device CSR builder
# ----------------------------------------------------------------------------------------

def csr_from_keys(n, keys, device="cuda"):
    """Directed keys (u<<32 | w, int64/uint64 tensor holding both directions) -> sorted,
    deduplicated, self-loop-free CSR on the device (symmetrize's contract, graph.py:452-481).
    ``keys`` is clobbered."""
    lib = _lib.load()
    keys = keys.contiguous()
    nk = keys.shape[0]
    alt = torch.empty_like(keys)
    off = torch.empty(n + 1, dtype=torch.int64, device=device)
    tgt = torch.empty(max(nk, 1), dtype=torch.int32, device=device)
    mdev = torch.empty(1, dtype=torch.int64, device=device)
    tb = lib.pasgal_csr_build_temp_bytes(n, nk)
    temp = torch.empty(tb, dtype=torch.uint8, device=device)
    st = lib.pasgal_csr_from_keys(n, _ptr(keys), _ptr(alt), nk, _ptr(off), _ptr(tgt), _ptr(mdev),
                                  _ptr(temp), tb, _stream(device))
    _lib.check(st, "csr_from_keys")
    m = _read_scalar(mdev)
    del alt, temp
    return DeviceGraph(off, tgt[:m])


def symmetrize_edges(n, src, dst, device="cuda"):
    """symmetrize(from_edges(n, src, dst)) on the device: both directions, self-loops
    dropped, duplicates removed, rows sorted (graph.py:452-481)."""
    s = torch.as_tensor(np.asarray(src, dtype=np.int64)).to(device)
    d = torch.as_tensor(np.asarray(dst, dtype=np.int64)).to(device)
    if s.shape != d.shape:
        raise ValueError("src/dst length mismatch")
    if s.numel() and (int(s.min()) < 0 or int(s.max()) >= n or int(d.min()) < 0 or int(d.max()) >= n):
        raise ValueError("edge endpoint out of range")
    keys = torch.cat([(s << 32) | d, (d << 32) | s])
    return csr_from_keys(n, keys, device)


# ----------------------------------------------------------------------------------------
# generators
# ----------------------------------------------------------------------------------------

def grid_threshold(p):
    """Edge kept iff draw < floor(p * 2^64); p >= 1 keeps the full lattice."""
    if p >= 1.0:
        return 0, 1
    if p < 0:
        raise ValueError("p must be >= 0")
    return int(float(p) * 2.0 ** 64), 0


def rmat_thresholds(a, b, c):
    s = 2.0 ** 32
    cap = 2 ** 32 - 1
    return min(int(a * s), cap), min(int((a + b) * s), cap), min(int((a + b + c) * s), cap)


def gen_grid(rows, cols, p=1.0, seed=0, device="cuda"):
    """rows x cols 4-neighbour lattice, each edge kept with probability p (seeded).
    p=1 reproduces the reference's gen_grid (graph.py:488-508, row-major ids)."""
    lib = _lib.load()
    if rows < 1 or cols < 1:
        raise ValueError("grid dimensions must be >= 1")
    n = rows * cols
    thr, keep_all = grid_threshold(p)
    off = torch.empty(n + 1, dtype=torch.int64, device=device)
    tgt = torch.empty(4 * n, dtype=torch.int32, device=device)
    mdev = torch.empty(1, dtype=torch.int64, device=device)
    tb = lib.pasgal_gen_grid_temp_bytes(rows, cols)
    temp = torch.empty(tb, dtype=torch.uint8, device=device)
    st = lib.pasgal_gen_grid(rows, cols, seed, thr, keep_all, _ptr(off), _ptr(tgt), _ptr(mdev),
                             _ptr(temp), tb, _stream(device))
    _lib.check(st, "gen_grid")
    m = _read_scalar(mdev)
    return DeviceGraph(off, tgt[:m].clone())


def gen_rmat(scale, draws, seed=1, a=0.57, b=0.19, c=0.19, device="cuda"):
    """RMAT on 2^scale vertices from `draws` seeded edge draws; self-loops dropped,
    duplicates removed, symmetrised (no vertex permutation)."""
    lib = _lib.load()
    ta, tab, tabc = rmat_thresholds(a, b, c)
    keys = torch.empty(max(2 * draws, 1), dtype=torch.int64, device=device)
    nk = torch.empty(1, dtype=torch.int64, device=device)
    st = lib.pasgal_gen_rmat_keys(scale, draws, seed, ta, tab, tabc, _ptr(keys), _ptr(nk), _stream(device))
    _lib.check(st, "gen_rmat")
    return csr_from_keys(1 << scale, keys[: 2 * draws], device)


def knn_gbits(npts):
    g = 0
    while g < 12 and (1 << (2 * (g + 1))) <= max(npts // 2, 1):
        g += 1
    return g


def gen_knn(npts, k=5, seed=1, device="cuda"):
    """k nearest neighbours of npts seeded points in the unit square (24-bit coordinates,
    exact integer distances, ties by index), symmetrised and deduplicated."""
    lib = _lib.load()
    g = knn_gbits(npts)
    keys = torch.empty(max(2 * k * npts, 1), dtype=torch.int64, device=device)
    nk = torch.empty(1, dtype=torch.int64, device=device)
    tb = lib.pasgal_gen_knn_temp_bytes(npts, g)
    temp = torch.empty(tb, dtype=torch.uint8, device=device)
    st = lib.pasgal_gen_knn_keys(npts, k, seed, g, _ptr(keys), _ptr(nk), _ptr(temp), tb, _stream(device))
    _lib.check(st, "gen_knn")
    del temp
    return csr_from_keys(npts, keys[: 2 * k * npts], device)


# BASELINE.json configs; seeds fixed at 1
CONFIGS = {
    "c1": dict(kind="grid", rows=256, cols=256, p=0.6, seed=1,
               desc="grid 256x256, p=0.6 (BASELINE configs[0])"),
    "c2": dict(kind="rmat", scale=20, draws=1 << 24, seed=1,
               desc="RMAT scale 20, 2^24 draws, (a,b,c,d)=(.57,.19,.19,.05) (configs[1])"),
    "c3": dict(kind="grid", rows=4096, cols=4096, p=0.6, seed=1,
               desc="grid 4096x4096, p=0.6 (configs[2])"),
    "c4": dict(kind="knn", npts=1 << 25, k=5, seed=1,
               desc="kNN k=5 on 2^25 uniform points (configs[3])"),
    "c5a": dict(kind="rmat", scale=28, draws=1 << 31, seed=1,
                desc="RMAT scale 28, 2^31 draws (avg degree 16) (configs[4a])"),
}


def make_config(name, device="cuda", seed=None, scale_override=None):
    """Generate a BASELINE config on the device.  ``seed`` overrides the config seed."""
    cfg = dict(CONFIGS[name])
    if seed is not None:
        cfg["seed"] = seed
    kind = cfg["kind"]
    if kind == "grid":
        return gen_grid(cfg["rows"], cfg["cols"], cfg["p"], cfg["seed"], device)
    if kind == "rmat":
        scale = scale_override or cfg["scale"]
        draws = cfg["draws"] >> (cfg["scale"] - scale) if scale_override else cfg["draws"]
        return gen_rmat(scale, draws, cfg["seed"], device=device)
    if kind == "knn":
        return gen_knn(cfg["npts"], cfg["k"], cfg["seed"], device)
    raise ValueError(kind)
