"""FAST-BCC entry points: the drop-in for the reference's BCC call.

``bcc(g)`` has the call shape of ``pasgal.oracles.bcc_hopcroft_tarjan(g)``
(oracles.py:119-201) and returns a ``BccLabels`` (results.py:45-88) that the reference's
``canonical_edge_partition`` (results.py:103-112) accepts unchanged.  The work runs on the
B200 through libpasgal_bcc.so (include/pasgal_bcc.h); there is no CPU fallback.

``bcc_device(offsets, targets)`` is the device-resident form: torch CUDA tensors in,
torch CUDA tensors out, stream-ordered on the current stream, no host synchronisation
unless ``validate=True``.
"""

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .graph import DeviceGraph
from .results import BccLabels

_ws_cache = {}


def _vp(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def workspace_bytes(n, m):
    return int(_lib.load().pasgal_bcc_workspace_bytes(int(n), int(m)))


def validate_workspace_bytes(n, m):
    return int(_lib.load().pasgal_csr_validate_workspace_bytes(int(n), int(m)))


def _workspace(device, nbytes, kind="bcc"):
    """A cached device workspace of at least nbytes (the library never allocates).
    ``kind`` separates buffers that are in use at the same time (BCC and validation)."""
    key = (kind, torch.device(device))
    ws = _ws_cache.get(key)
    if ws is None or ws.numel() < nbytes:
        _ws_cache.pop(key, None)
        ws = torch.empty(int(nbytes), dtype=torch.uint8, device=key[1])
        _ws_cache[key] = ws
    return ws


def release_workspace():
    _graphs.clear()
    _ws_cache.clear()
    _side_streams.clear()
    _priority_streams.clear()


_side_streams = {}


def _side_stream(device):
    dev = torch.device(device)
    if dev not in _side_streams:
        _side_streams[dev] = torch.cuda.Stream(dev, priority=0)    # 0 = the lowest priority
    return _side_streams[dev]


class _PendingValidation:
    """Second half of a split validation (pasgal_csr_validate_end): the symmetry check,
    run on the side stream after `after` (an event: the BCC kernels) so it overlaps
    whatever follows them on the main stream (the labels' D2H copy)."""

    def __init__(self, csr, ws, stream, keep):
        self.csr, self.ws, self.stream, self.keep = csr, ws, stream, keep

    def finish(self, after=None):
        if after is not None:
            self.stream.wait_event(after)
        st = _lib.load().pasgal_csr_validate_end(ctypes.byref(self.csr), _vp(self.ws), self.ws.numel(),
                                                 ctypes.c_void_p(self.stream.cuda_stream))
        self.keep = None
        _lib.check(st, "validate")


def _validate_begin(offsets, targets, ws=None, side=None):
    """Run the blocking streaming checks now (ranges, row order, up/down balance: after
    this the CSR is safe for FAST-BCC); the symmetry check is the returned object's
    finish().  Raises at once on an early failure."""
    lib = _lib.load()
    dev = offsets.device
    n, m = offsets.shape[0] - 1, targets.shape[0]
    if ws is None:
        ws = _workspace(dev, validate_workspace_bytes(n, m), kind="validate")
    if side is None:
        side = _side_stream(dev)
    side.wait_stream(torch.cuda.current_stream(dev))        # the CSR's H2D copies
    csr = _csr_struct(offsets, targets)
    st = lib.pasgal_csr_validate_begin(ctypes.byref(csr), _vp(ws), ws.numel(), ctypes.c_void_p(side.cuda_stream))
    _lib.check(st, "validate")
    return _PendingValidation(csr, ws, side, (offsets, targets))


@dataclass
class DeviceBcc:
    """Device outputs of one BCC run."""

    edge_label: torch.Tensor    # int32 storage of uint32 labels [M] (0xFFFFFFFF = none)
    artic_bits: torch.Tensor    # int32 storage of the uint32 bitmap [ceil(n/32)]
    bcc_count: torch.Tensor     # int64 [1]
    comp: torch.Tensor = None   # optional int32 [n]
    parent: torch.Tensor = None
    first: torch.Tensor = None
    launches: int = 0           # kernel launches the call issued


def _csr_struct(offsets, targets):
    n = offsets.shape[0] - 1
    m = targets.shape[0]
    return _lib.PasgalCsr(n, m, offsets.data_ptr(), targets.data_ptr() if m else 0)


def validate_device(offsets, targets, workspace=None):
    """Device check of the BCC preconditions (symmetric, sorted rows, ids in range).
    Synchronises; raises ValueError like the reference (oracles.py:127-128).  A given
    ``workspace`` smaller than ``validate_workspace_bytes(n, m)`` is replaced by the cached
    one (validation needs O(m) scratch, the BCC workspace only O(n))."""
    lib = _lib.load()
    n, m = offsets.shape[0] - 1, targets.shape[0]
    need = validate_workspace_bytes(n, m)
    ws = (workspace if workspace is not None and workspace.numel() >= need
          else _workspace(offsets.device, need, kind="validate"))
    csr = _csr_struct(offsets, targets)
    st = lib.pasgal_csr_validate(ctypes.byref(csr), _vp(ws), ws.numel(),
                                 ctypes.c_void_p(torch.cuda.current_stream(offsets.device).cuda_stream))
    _lib.check(st, "validate")


GRAPH_MAX_N = 1 << 26       # auto CUDA-graph replay below this size (launch gaps matter up to C4)
_GRAPH_CACHE_SIZE = 8


class _GraphCache:
    """Captured pasgal_bcc calls (pasgal_bcc_graph_create), keyed by every pointer, size,
    seed and flag they were captured with, least recently used evicted first."""

    def __init__(self):
        self.entries = {}

    def get(self, key, create):
        h = self.entries.pop(key, None)
        if h is None:
            h = create()
            while len(self.entries) >= _GRAPH_CACHE_SIZE:
                old = next(iter(self.entries))
                _lib.load().pasgal_bcc_graph_destroy(self.entries.pop(old))
        self.entries[key] = h
        return h

    def clear(self):
        lib = _lib.load() if self.entries else None
        for h in self.entries.values():
            lib.pasgal_bcc_graph_destroy(h)
        self.entries.clear()


_graphs = _GraphCache()


def bcc_device(offsets, targets, *, seed=0, validate=False, canonical=False, out=None,
               workspace=None, forest=False, edge_labels=True, events=None, graph=None,
               _defer_validation=False):
    """FAST-BCC on a device CSR (offsets int64[n+1], targets int32[M], both CUDA).

    Returns ``DeviceBcc``.  ``canonical=True`` labels every edge with the minimum
    undirected edge id of its BCC.  ``forest=True`` also returns comp/parent/first (the
    parallel-mode fields of BccLabels).  ``edge_labels=False`` (vertex mode, implies
    ``forest``) skips the per-slot labelling pass: the result is O(n) sized
    (results.py:49-52) and ``edge_label`` is None.  ``events``: optional list of
    ``torch.cuda.Event(enable_timing=True)`` (one per stage, ``_lib.STAGES``) recorded at
    the stage boundaries on the current stream.  ``graph``: replay a captured CUDA graph of
    the call (pasgal_bcc_graph_*; cached per pointer/size/seed/flags set).  The default
    (None) does so for graphs below GRAPH_MAX_N vertices when the caller passes both
    ``out`` and ``workspace`` (fixed buffers: a repeated call), without ``events``."""
    lib = _lib.load()
    if offsets.device.type != "cuda" or targets.device.type != "cuda":
        raise ValueError("bcc_device needs CUDA tensors")
    if offsets.dtype != torch.int64 or targets.dtype != torch.int32:
        raise ValueError("offsets must be int64 and targets int32")
    offsets = offsets.contiguous()
    targets = targets.contiguous()
    n, m = offsets.shape[0] - 1, targets.shape[0]
    dev = offsets.device
    need = workspace_bytes(n, m)
    ws = workspace if workspace is not None else _workspace(dev, need)
    if ws.numel() < need:
        raise ValueError("workspace too small")
    if not edge_labels:
        if canonical:
            raise ValueError("canonical labels need edge_labels=True")
        forest = True
    # validation is split: its streaming half gates the call, its symmetry half runs after
    # the BCC kernels on a side stream (overlapping the caller's next copies when deferred)
    pending = _validate_begin(offsets, targets) if validate else None
    if out is None:
        out = DeviceBcc(
            edge_label=torch.empty(m, dtype=torch.int32, device=dev) if edge_labels else None,
            artic_bits=torch.empty((n + 31) // 32, dtype=torch.int32, device=dev),
            bcc_count=torch.empty(1, dtype=torch.int64, device=dev),
        )
        if forest:
            out.comp = torch.empty(n, dtype=torch.int32, device=dev)
            out.parent = torch.empty(n, dtype=torch.int32, device=dev)
            out.first = torch.empty(n, dtype=torch.int32, device=dev)
    csr = _csr_struct(offsets, targets)
    if not edge_labels and (out.comp is None or out.parent is None or out.first is None):
        raise ValueError("vertex mode needs out.comp, out.parent and out.first")
    o = _lib.PasgalBccOut(out.edge_label.data_ptr() if (m and edge_labels and out.edge_label is not None) else 0, out.artic_bits.data_ptr() if n else 0,
                          out.bcc_count.data_ptr(),
                          out.comp.data_ptr() if out.comp is not None else 0,
                          out.parent.data_ptr() if out.parent is not None else 0,
                          out.first.data_ptr() if out.first is not None else 0)
    flags = _lib.PASGAL_BCC_CANONICAL if canonical else 0
    stream = torch.cuda.current_stream(dev)
    prof = _lib.PasgalBccProf(None, 0, 0)
    if events is not None:
        handles = []
        for e in events:
            if e.cuda_event == 0:       # torch creates the event lazily on first record
                e.record(stream)
            handles.append(e.cuda_event)
        arr = (ctypes.c_void_p * len(handles))(*handles)
        prof = _lib.PasgalBccProf(ctypes.cast(arr, ctypes.POINTER(ctypes.c_void_p)), len(handles), 0)
    if graph is None:
        graph = events is None and workspace is not None and out is not None and n < GRAPH_MAX_N
    if graph and events is None:
        key = (dev, offsets.data_ptr(), targets.data_ptr(), n, m, o.edge_label, o.artic_bits, o.bcc_count, o.comp,
               o.parent, o.first, ws.data_ptr(), ws.numel(), int(seed) & (2**64 - 1), flags)

        def create():
            h = ctypes.c_void_p()
            _lib.check(lib.pasgal_bcc_graph_create(ctypes.byref(csr), ctypes.byref(o), _vp(ws), ws.numel(),
                                                   int(seed) & (2**64 - 1), flags, ctypes.byref(h)), "bcc graph")
            return h

        nl = ctypes.c_int(0)
        st = lib.pasgal_bcc_graph_launch(_graphs.get(key, create), ctypes.c_void_p(stream.cuda_stream),
                                         ctypes.byref(nl))
        prof.launches = nl.value
    else:
        st = lib.pasgal_bcc_ex(ctypes.byref(csr), ctypes.byref(o), _vp(ws), ws.numel(), int(seed) & (2**64 - 1),
                               flags, ctypes.c_void_p(stream.cuda_stream), ctypes.byref(prof))
    if st != 0 and pending is not None:
        pending.finish()            # a symmetry error explains a failure better
    _lib.check(st, "bcc")
    out.launches = prof.launches
    if pending is not None:
        if _defer_validation:
            return out, pending
        pending.finish()
    return out


def connected_components_device(offsets, targets, *, seed=0, workspace=None):
    """Connected components of a symmetric device CSR: returns
    (comp int32 tensor [n] holding each vertex's component minimum id, count tensor)."""
    lib = _lib.load()
    offsets = offsets.contiguous()
    targets = targets.contiguous()
    n, m = offsets.shape[0] - 1, targets.shape[0]
    dev = offsets.device
    need = workspace_bytes(n, m)
    ws = workspace if workspace is not None else _workspace(dev, need)
    comp = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    count = torch.empty(1, dtype=torch.int64, device=dev)
    csr = _csr_struct(offsets, targets)
    st = lib.pasgal_cc(ctypes.byref(csr), _vp(comp), _vp(count), _vp(ws), ws.numel(), int(seed) & (2**64 - 1),
                       ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream))
    _lib.check(st, "cc")
    return comp[:n], count


def connected_components(g, *, seed=0, validate=True, device="cuda"):
    """Host form: (labels int64[n] = component minimum vertex id, component count)."""
    if isinstance(g, DeviceGraph):
        off_d, tgt_d = g.offsets, g.targets
    else:
        off_d = torch.from_numpy(np.ascontiguousarray(g.offsets, dtype=np.int64)).to(device)
        tg = np.asarray(g.targets)
        tg = tg.view(np.int32) if tg.dtype == np.uint32 else tg.astype(np.int32)
        tgt_d = torch.from_numpy(np.ascontiguousarray(tg)).to(device)
    if validate:
        validate_device(off_d, tgt_d)
    comp, count = connected_components_device(off_d, tgt_d, seed=seed)
    return comp.cpu().numpy().astype(np.int64), int(count.item())


def canonicalize_device(offsets, targets, labels, label_bound=None):
    """Device canonical form of any per-slot labelling (results.py:91-112 semantics): every
    slot gets the minimum undirected edge id of its class.  ``labels``: int32/uint32 CUDA
    tensor with ids in [0, label_bound) (default: max(n, M)); 0xFFFFFFFF passes through."""
    lib = _lib.load()
    offsets = offsets.contiguous()
    targets = targets.contiguous()
    n, m = offsets.shape[0] - 1, targets.shape[0]
    bound = int(label_bound if label_bound is not None else max(n, m, 1))
    lab = labels.contiguous().view(torch.int32)
    out = torch.empty_like(lab)
    tb = lib.pasgal_canonicalize_temp_bytes(n, m, bound)
    temp = torch.empty(tb, dtype=torch.uint8, device=offsets.device)
    csr = _csr_struct(offsets, targets)
    st = lib.pasgal_canonicalize(ctypes.byref(csr), _vp(lab), bound, _vp(out), _vp(temp), tb,
                                 ctypes.c_void_p(torch.cuda.current_stream(offsets.device).cuda_stream))
    _lib.check(st, "canonicalize")
    return out


def canonical_checksum_device(canon_labels, artic_bits, bcc_count):
    """Device twin of results.canonical_checksum (pasgal_canonical_checksum: one pass, no
    M-sized temporaries): canon_labels is the int32 storage of the canonical uint32 labels
    (bcc_device(..., canonical=True).edge_label), artic_bits the device bitmap, bcc_count
    the device count.  Products and sums wrap mod 2^64 exactly as the host's uint64 ones."""
    m = canon_labels.shape[0]
    nw = artic_bits.shape[0]
    out = torch.empty(2, dtype=torch.int64, device=canon_labels.device)
    st = _lib.load().pasgal_canonical_checksum(_vp(canon_labels.contiguous()), int(m), _vp(artic_bits.contiguous()),
                                                int(32 * nw), _vp(out),
                                                ctypes.c_void_p(torch.cuda.current_stream(canon_labels.device).cuda_stream))
    _lib.check(st, "checksum")
    h, nart = (int(x) for x in out.cpu().tolist())
    return int(bcc_count.item()), nart, h % (1 << 64)


def same_partition_device(offsets, targets, labels_a, labels_b, label_bound=None):
    """True iff two per-slot labellings induce the same edge partition (device comparator)."""
    a = canonicalize_device(offsets, targets, labels_a, label_bound)
    b = canonicalize_device(offsets, targets, labels_b, label_bound)
    return bool(torch.equal(a, b))


def unpack_articulation(bits, n):
    """uint32 bitmap (bit v&31 of word v>>5) -> bool[n]."""
    b = np.ascontiguousarray(bits).view(np.uint8)
    return np.unpackbits(b, bitorder="little")[:n].astype(bool)


def articulation_bytes_device(bits, n):
    """Device uint32 bitmap -> device uint8[n] (0/1), by the library's kernel."""
    out = torch.empty(max(n, 1), dtype=torch.uint8, device=bits.device)
    st = _lib.load().pasgal_bits_to_bytes(_vp(bits), int(n), _vp(out),
                                          ctypes.c_void_p(torch.cuda.current_stream(bits.device).cuda_stream))
    _lib.check(st, "bits_to_bytes")
    return out[:n]


@dataclass
class HostBuffers:
    """Optional caller-owned (ideally pinned) host buffers for ``bcc(..., host_out=)``:
    labels and articulation flags are copied straight into them and the returned
    BccLabels views them (no host-side copy or unpack)."""

    edge_label: torch.Tensor    # int32 [>= M], cpu (pinned); None in vertex mode
    articulation: torch.Tensor  # uint8 [>= n], cpu (pinned)
    comp: torch.Tensor = None   # int32 [>= n] each, vertex mode (edge_labels=False)
    parent: torch.Tensor = None
    first: torch.Tensor = None

    @staticmethod
    def allocate(n, m, pinned=True, edge_labels=True):
        def buf(k, dt):
            return torch.empty(max(k, 1), dtype=dt, pin_memory=pinned)

        if edge_labels:
            return HostBuffers(buf(m, torch.int32), buf(n, torch.uint8))
        return HostBuffers(None, buf(n, torch.uint8), buf(n, torch.int32), buf(n, torch.int32), buf(n, torch.int32))


def bcc(g, *, seed=0, validate=True, canonical=False, device="cuda", forest=False, host_out=None,
        edge_labels=True):
    """Drop-in for ``bcc_hopcroft_tarjan(g)``: biconnected components of a symmetric graph.

    ``g`` is any object with ``offsets`` (int64[n+1]) and ``targets`` (uint32/int32/int64
    [M]) -- a pasgal Graph, this package's Graph, or a DeviceGraph.  The CSR is copied to
    the device, validated there (``ValueError("biconnectivity requires a symmetric graph")``
    as in oracles.py:127-128), processed, and the labels, articulation flags and count are
    copied back into a ``BccLabels``.  Rows must be sorted (every reference builder sorts).

    ``edge_labels=False`` returns the reference's O(n) parallel-mode ``BccLabels``
    (comp/parent/first, results.py:49-52, 76-88) instead of per-slot labels: the device
    skips the labelling pass and the copy back is 13 bytes per vertex instead of 4 per slot;
    ``edge_labels(g)`` derives the per-slot labels on the host on demand.

    The work runs on a high-priority stream: the validation's symmetry check, on the
    lowest-priority side stream, then only fills the SMs the BCC kernels leave idle
    instead of delaying them (its ~8M-block grid would otherwise be dispatched first).
    """
    dev = torch.device(device) if not isinstance(g, DeviceGraph) else g.offsets.device
    if dev.type == "cuda" and dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    cur = torch.cuda.current_stream(dev)
    hp = _priority_stream(dev)
    hp.wait_stream(cur)
    with torch.cuda.stream(hp):
        res = _bcc_host(g, seed, validate, canonical, device, forest, host_out, edge_labels)
    cur.wait_stream(hp)
    return res


_priority_streams = {}


def _priority_stream(device):
    if device not in _priority_streams:
        # torch maps an out-of-range priority to the nearest valid one: the greatest here
        _priority_streams[device] = torch.cuda.Stream(device, priority=-100)
    return _priority_streams[device]


def _bcc_host(g, seed, validate, canonical, device, forest, host_out, edge_labels=True):
    if isinstance(g, DeviceGraph):
        off_d, tgt_d = g.offsets, g.targets
    else:
        off = np.ascontiguousarray(g.offsets, dtype=np.int64)
        tgt = np.asarray(g.targets)
        n_host = off.shape[0] - 1
        if n_host >= 2 ** 31 or tgt.shape[0] >= 2 ** 32:
            raise ValueError("graph too large for int32 vertex ids / uint32 slot ids")
        if tgt.dtype == np.uint32:
            tgt = tgt.view(np.int32)
        elif tgt.dtype != np.int32:
            if tgt.shape[0] and (int(tgt.max()) >= n_host or int(tgt.min()) < 0):
                raise ValueError("edge target out of range")
            tgt = tgt.astype(np.int32)
        tgt = np.ascontiguousarray(tgt)
        off_d = torch.from_numpy(off).to(device, non_blocking=True)
        tgt_d = torch.from_numpy(tgt).to(device, non_blocking=True)
    n = off_d.shape[0] - 1
    m = tgt_d.shape[0]
    r = bcc_device(off_d, tgt_d, seed=seed, validate=validate, canonical=canonical, forest=forest,
                   edge_labels=edge_labels, _defer_validation=validate)
    pending = None
    if validate:
        r, pending = r
    art_d = articulation_bytes_device(r.artic_bits, n)
    done = torch.cuda.Event()
    done.record()                           # BCC kernels + articulation bytes
    if not edge_labels:
        hb = host_out if host_out is not None else HostBuffers.allocate(n, m, edge_labels=False)
        fields = []
        for src, dst in ((art_d, hb.articulation), (r.comp, hb.comp), (r.parent, hb.parent), (r.first, hb.first)):
            dst[:n].copy_(src[:n], non_blocking=True)
            fields.append(dst[:n].numpy())
        if pending is not None:
            pending.finish(after=done)
        count = int(r.bcc_count.item())     # synchronises the stream
        art, comp, par, fst = fields
        return BccLabels(art.view(np.bool_), count, comp=comp.view(np.uint32), parent=par.view(np.uint32),
                         first=fst.view(np.uint32))
    if host_out is not None:
        host_out.edge_label[:m].copy_(r.edge_label, non_blocking=True)
        host_out.articulation[:n].copy_(art_d, non_blocking=True)
        if pending is not None:
            pending.finish(after=done)      # the symmetry check runs during the D2H above
        count = int(r.bcc_count.item())     # synchronises the stream
        lab = host_out.edge_label[:m].numpy().view(np.uint32)
        art = host_out.articulation[:n].numpy().view(np.bool_)
    else:
        if pending is not None:
            pending.finish(after=done)
        lab = r.edge_label.cpu().numpy().view(np.uint32)
        art = art_d.cpu().numpy().view(np.bool_)
        count = int(r.bcc_count.item())
    if forest:
        return BccLabels(art, count, edge_label=lab,
                         comp=r.comp.cpu().numpy().astype(np.int64),
                         parent=r.parent.cpu().numpy().astype(np.int64),
                         first=r.first.cpu().numpy().astype(np.int64))
    return BccLabels(art, count, edge_label=lab)
