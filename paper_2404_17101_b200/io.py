"""Graph files -> device CSR: the binary layout of the reference's
load_bin / save_bin (graph.py:360-409; GBBS-style: u64 n, u64 m, u64 size, (n+1) u64
offsets, m u32 targets).

``load_bin`` memory-maps the file, checks the header on the host and raises
``GraphFormatError`` (a ValueError carrying path and byte position, as graph.py:31-46) for
truncation and size-field mismatches; the offset and target arrays go straight to HBM
and their range checks run on the device, which reports the first offending index so the
error names the same byte position the reference would.  The BCC path is unweighted:
a ``.wbin`` file's trailing weight block is validated for length and ignored.
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
    return DeviceGraph(off, tgt)


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
