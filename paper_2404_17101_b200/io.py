"""Graph files -> device CSR: the binary layout of the reference's
load_bin / save_bin (graph.py:360-409; GBBS-style: u64 n, u64 m, u64 size, (n+1) u64
offsets, m u32 targets) and its text adjacency format load_adj / save_adj
(graph.py:250-336).

``load_bin`` memory-maps the file, checks the header on the host and raises
``GraphFormatError`` (a ValueError carrying path and byte position, as graph.py:31-46) for
truncation and size-field mismatches; the offset and target arrays go straight to HBM
and their range checks run on the device, which reports the first offending index so the
error names the same byte position the reference would.  The BCC path is unweighted:
a ``.wbin`` file's trailing weight block is validated (length, and the reference's
negative-weight error, graph.py:384-390, checked on the device) and not returned.
``load_graph`` dispatches on the extension like graph.py:411-418.
"""

import ctypes
import struct
from pathlib import Path

import numpy as np
import torch

from . import _lib
from .graph import DeviceGraph

_HDR = 24


class GraphFormatError(ValueError):
    """Malformed graph file; carries the offending position (graph.py:31-46)."""

    def __init__(self, message, path=None, line=None, byte=None):
        where = [str(x) for x in (path,) if x is not None]
        if line is not None:
            where.append(f"line {line}")
        if byte is not None:
            where.append(f"byte {byte}")
        super().__init__(message + (f" ({', '.join(where)})" if where else ""))
        self.path, self.line, self.byte = path, line, byte


def load_bin(path, device="cuda"):
    path = Path(path)
    size = path.stat().st_size
    if size < _HDR:
        raise GraphFormatError(f"truncated file: {size} bytes, need >= {_HDR}", path, byte=size)
    mm = np.memmap(path, dtype=np.uint8, mode="r")
    n, m, size_field = struct.unpack_from("<QQQ", mm[:_HDR].tobytes(), 0)
    if n >= 2 ** 31:
        raise GraphFormatError(f"vertex count {n} exceeds the int32 vertex ids of the device CSR", path, byte=0)
    if m >= 2 ** 32:
        raise GraphFormatError(f"edge count {m} exceeds the uint32 slot ids of the device CSR", path, byte=8)
    base = _HDR + (n + 1) * 8 + m * 4
    if size_field != base:
        raise GraphFormatError(f"size-field mismatch: header says {size_field}, layout needs {base}", path, byte=16)
    need = base + (m * 4 if path.suffix == ".wbin" else 0)
    if size < need:
        raise GraphFormatError(f"truncated file: {size} bytes, need {need}", path, byte=size)
    off_np = np.frombuffer(mm, dtype="<u8", count=n + 1, offset=_HDR)
    if int(off_np[0]) != 0 or int(off_np[-1]) != m:
        raise GraphFormatError(f"offset block invalid: first={int(off_np[0])} last={int(off_np[-1])} m={m}",
                               path, byte=_HDR)
    tgt_np = np.frombuffer(mm, dtype="<u4", count=m, offset=_HDR + (n + 1) * 8)
    off = torch.from_numpy(off_np.view(np.int64).copy()).to(device)
    tgt = torch.from_numpy(tgt_np.view(np.int32).copy()).to(device) if m else torch.empty(0, dtype=torch.int32,
                                                                                           device=device)
    # array checks on the device, positioned like the reference's messages
    lib = _lib.load()
    csr = _lib.PasgalCsr(n, m, off.data_ptr(), tgt.data_ptr() if m else 0)
    res = (ctypes.c_int64 * 2)()
    scratch = torch.empty(2, dtype=torch.int64, device=off.device)
    _lib.check(lib.pasgal_csr_first_error(ctypes.byref(csr), ctypes.c_void_p(scratch.data_ptr()), res,
                                          ctypes.c_void_p(torch.cuda.current_stream(off.device).cuda_stream)),
               "load_bin")
    if res[0] >= 0:
        i = int(res[0])
        raise GraphFormatError(f"offsets decrease at index {i}", path, byte=_HDR + i * 8)
    if res[1] >= 0:
        i = int(res[1])
        t = int(tgt_np[i])
        raise GraphFormatError(f"target out of range at edge {i}: {t} >= n={n}", path,
                               byte=_HDR + (n + 1) * 8 + i * 4)
    if path.suffix == ".wbin" and m:
        # graph.py:384-390 tests weights.min() < 0: -0.0 passes, and numpy's min propagates
        # NaN, so a block holding any NaN passes whatever else it holds
        w = torch.from_numpy(np.frombuffer(mm, dtype="<f4", count=m, offset=base).copy()).to(device)
        neg = torch.nonzero(w < 0)
        if neg.numel() and not bool(torch.isnan(w).any().item()):
            i = int(neg[0, 0].item())
            raise GraphFormatError(f"negative weight at edge {i}", path, byte=base + i * 4)
    return DeviceGraph(off, tgt)


def load_graph(path, weighted=None, device="cuda"):
    """Dispatch on extension (graph.py:411-418): .adj -> load_adj, .bin/.wbin -> load_bin."""
    p = Path(path)
    if p.suffix == ".adj":
        return load_adj(p, weighted, device=device)
    if p.suffix in (".bin", ".wbin"):
        return load_bin(p, device=device)
    raise GraphFormatError(f"unknown graph extension {p.suffix!r}", p)


ADJ_HEADER = b"AdjacencyGraph"
WADJ_HEADER = b"WeightedAdjacencyGraph"
_WS_CODES = np.frombuffer(b" \t\n\r\x0b\x0c", dtype=np.uint8)
_OVERFLOW = "Python int too large to convert to C long"   # numpy's int64 conversion error


class _AdjText:
    """Raw file bytes on the device plus the tokenizer state (csrc/adj.cu)."""

    def __init__(self, raw, device):
        self.raw = raw
        self.L = int(raw.shape[0])
        self.lib = _lib.load()
        self.text = (torch.from_numpy(raw).to(device) if self.L else torch.empty(16, dtype=torch.uint8, device=device))
        self.temp = torch.empty(int(self.lib.pasgal_adj_temp_bytes(self.L)), dtype=torch.uint8, device=device)
        self.stream = ctypes.c_void_p(torch.cuda.current_stream(self.text.device).cuda_stream)
        nt = ctypes.c_int64()
        _lib.check(self.lib.pasgal_adj_tokenize(self._p(self.text), self.L, self._p(self.temp), self.temp.numel(),
                                                ctypes.byref(nt), self.stream), "load_adj")
        self.ntokens = nt.value

    @staticmethod
    def _p(t):
        return ctypes.c_void_p(t.data_ptr())

    def position(self, k):
        """(line, byte) of token k, as the reference's _token_position (graph.py:200-214)."""
        bl = (ctypes.c_int64 * 2)()
        _lib.check(self.lib.pasgal_adj_token_position(self._p(self.text), self.L, self._p(self.temp),
                                                      self.temp.numel(), int(k), bl, self.stream), "load_adj")
        return int(bl[1]), int(bl[0])

    def token(self, k):
        """Bytes of token k, read from the host copy of the file."""
        b = e = self.position(k)[1]
        while e < self.L:
            chunk = self.raw[e:e + 4096]
            hit = np.flatnonzero(np.isin(chunk, _WS_CODES))
            if hit.size:
                e += int(hit[0])
                break
            e += chunk.shape[0]
        return bytes(self.raw[b:e])


def _int_block(tokens, what, first_index, adj, path):
    """The reference's _parse_int_block (graph.py:217-230) on a few host tokens."""
    try:
        return np.array(tokens, dtype=np.int64)
    except (ValueError, OverflowError):
        for i, t in enumerate(tokens):
            try:
                int(t)
            except ValueError:
                raise GraphFormatError(f"invalid {what} token {t[:32]!r}", path,
                                       *adj.position(first_index + i)) from None
        raise


def load_adj(path, weighted=None, device="cuda"):
    """Load a text adjacency-graph file into a DeviceGraph (graph.py:250-318).

    Tokenizing and number parsing run on the device (csrc/adj.cu); only the header and the
    two count tokens are read on the host.  Errors reproduce the reference's checks in its
    order, with its messages and (line, byte) positions.  The BCC path is unweighted: a
    WeightedAdjacencyGraph's weights are validated as the reference does, then dropped."""
    path = Path(path)
    raw = np.fromfile(path, dtype=np.uint8)
    adj = _AdjText(raw, device)
    T = adj.ntokens
    if T == 0:
        raise GraphFormatError("empty file, missing header", path, 1, 0)
    header = adj.token(0)
    if header not in (ADJ_HEADER, WADJ_HEADER):
        raise GraphFormatError(f"malformed header {header[:40]!r}", path, 1, 0)
    has_w = header == WADJ_HEADER
    if weighted is not None and weighted != has_w:
        raise GraphFormatError(f"header {header.decode()} does not match weighted={weighted}", path, 1, 0)
    if T < 3:
        raise GraphFormatError("missing vertex/edge counts", path, *adj.position(T))
    counts = _int_block([adj.token(1), adj.token(2)], "count", 1, adj, path)
    n, m = int(counts[0]), int(counts[1])
    if n < 0 or m < 0:
        raise GraphFormatError(f"negative counts n={n} m={m}", path, *adj.position(1))
    expected = 3 + n + m + (m if has_w else 0)
    if T != expected:
        raise GraphFormatError(f"token count mismatch: expected {expected}, found {T}", path,
                               *adj.position(min(T, expected)))
    if n >= 2 ** 31 or m >= 2 ** 32:
        raise GraphFormatError(f"graph too large for the device CSR (n={n}, m={m}): int32 ids, uint32 slots", path)
    off = torch.empty(n + 1, dtype=torch.int64, device=adj.text.device)
    tgt = torch.empty(max(m, 1), dtype=torch.int32, device=adj.text.device)
    err = (ctypes.c_int64 * _ADJ_NERR)()
    unc = (ctypes.c_int64 * _ADJ_UNC_CAP)()
    nunc = ctypes.c_int64()
    _lib.check(adj.lib.pasgal_adj_parse(adj._p(adj.text), adj.L, adj._p(adj.temp), adj.temp.numel(), n, m,
                                        int(has_w), adj._p(off), adj._p(tgt), err, unc, ctypes.byref(nunc),
                                        adj.stream), "load_adj")
    # offsets block: parse errors, then first == 0, range, order (graph.py:284-301)
    if err[_INV_OFF] >= 0:
        k = 3 + err[_INV_OFF]
        raise GraphFormatError(f"invalid offset token {adj.token(k)[:32]!r}", path, *adj.position(k))
    if err[_OVF_OFF] >= 0:
        raise OverflowError(_OVERFLOW)
    if n:
        if int(off[0].item()) != 0:
            raise GraphFormatError("first offset must be 0", path, *adj.position(3))
        i = err[_RNG_OFF]
        if i < 0 and n > 1:
            i = _first_decrease(off, n, m)
        if i >= 0:
            raise GraphFormatError(f"offset out of range at index {i}: {int(off[i].item())}", path,
                                   *adj.position(3 + i))
    # targets block (graph.py:303-310)
    if err[_INV_TGT] >= 0:
        k = 3 + n + err[_INV_TGT]
        raise GraphFormatError(f"invalid target token {adj.token(k)[:32]!r}", path, *adj.position(k))
    if err[_OVF_TGT] >= 0:
        raise OverflowError(_OVERFLOW)
    if err[_RNG_TGT] >= 0:
        i = err[_RNG_TGT]
        k = 3 + n + i
        raise GraphFormatError(f"target out of range at edge {i}: {int(adj.token(k))} >= n={n}", path,
                               *adj.position(k))
    # weights block (graph.py:312-318): checked, then dropped
    if has_w and m:
        if err[_INV_W] >= 0:
            k = 3 + n + m + err[_INV_W]
            raise GraphFormatError(f"invalid weight token {adj.token(k)[:32]!r}", path, *adj.position(k))
        bad = [err[_BAD_W]] if err[_BAD_W] >= 0 else []
        if nunc.value > _ADJ_UNC_CAP:           # pathological: decide every weight on the host
            ws = np.array(bytes(raw).split()[3 + n + m:], dtype=np.float64)
            bad += np.flatnonzero(~(ws >= 0)).tolist()[:1]
        else:
            bad += [int(unc[j]) for j in range(nunc.value) if not float(adj.token(3 + n + m + unc[j])) >= 0]
        if bad:
            i = min(bad)
            raise GraphFormatError(f"negative or invalid weight at edge {i}", path, *adj.position(3 + n + m + i))
    return DeviceGraph(off, tgt[:m])


_INV_OFF, _OVF_OFF, _RNG_OFF, _INV_TGT, _OVF_TGT, _RNG_TGT, _INV_W, _BAD_W = range(8)
_ADJ_NERR = 8
_ADJ_UNC_CAP = 1024


def _first_decrease(off, n, m):
    """First i >= 1 with offsets[i] < offsets[i-1] (device, via pasgal_csr_first_error)."""
    lib = _lib.load()
    csr = _lib.PasgalCsr(n, 0, off.data_ptr(), 0)
    res = (ctypes.c_int64 * 2)()
    scratch = torch.empty(2, dtype=torch.int64, device=off.device)
    _lib.check(lib.pasgal_csr_first_error(ctypes.byref(csr), ctypes.c_void_p(scratch.data_ptr()), res,
                                          ctypes.c_void_p(torch.cuda.current_stream(off.device).cuda_stream)),
               "load_adj")
    return int(res[0])


def save_adj(g, path):
    """Write the canonical text serialization (graph.py:321-336) of an unweighted graph."""
    path = Path(path)
    off = g.offsets.cpu().numpy() if isinstance(g.offsets, torch.Tensor) else np.asarray(g.offsets)
    tgt = g.targets.cpu().numpy() if isinstance(g.targets, torch.Tensor) else np.asarray(g.targets)
    n, m = off.shape[0] - 1, tgt.shape[0]
    chunks = [ADJ_HEADER, str(n).encode(), str(m).encode()]
    if n:
        chunks.append("\n".join(map(str, off[:-1].astype(np.int64).tolist())).encode())
    if m:
        chunks.append("\n".join(map(str, tgt.astype(np.int64).tolist())).encode())
    path.write_bytes(b"\n".join(chunks) + b"\n")


def save_bin(g, path):
    """Write the binary serialization (graph.py:398-409 layout) of an unweighted graph."""
    path = Path(path)
    off = g.offsets.cpu().numpy() if isinstance(g.offsets, torch.Tensor) else np.asarray(g.offsets)
    tgt = g.targets.cpu().numpy() if isinstance(g.targets, torch.Tensor) else np.asarray(g.targets)
    n, m = off.shape[0] - 1, tgt.shape[0]
    with open(path, "wb") as f:
        f.write(struct.pack("<QQQ", n, m, _HDR + (n + 1) * 8 + m * 4))
        f.write(off.astype("<u8").tobytes())
        f.write(tgt.astype("<u4").tobytes())
