"""Streamed BCC over many host graphs: the copies of one graph overlap the work of others.

``BccPipeline.run(graphs)`` yields one ``BccLabels`` per input graph, in order, with the same
contract as ``bcc(g)`` (validation included).  Three CUDA streams and two-slot device rings
keep the PCIe link busy in both directions:

* copy-in stream: H2D of graph i+1's CSR into input slot (i+1) % 2, once graph i-1's BCC and
  symmetry check have released that slot;
* compute stream (high priority): the streaming validation checks, FAST-BCC and the
  articulation bytes of graph i, into output slot i % 2 once graph i-2's D2H has drained it;
* copy-out stream: D2H of graph i's labels, articulation bytes and count into pinned host
  buffers (a two-slot host ring: a yielded result stays valid until the next is requested).

The symmetry half of the validation runs on the low-priority side stream after graph i's BCC
kernels, i.e. under its D2H, exactly as in ``bcc(g)``.  In steady state a step costs about
max(H2D, D2H, compute) instead of their sum.
"""

import ctypes

import numpy as np
import torch

from . import _lib
from .bcc import (_priority_stream, _validate_begin, _vp, _workspace, articulation_bytes_device,
                  validate_workspace_bytes, workspace_bytes)
from .graph import DeviceGraph
from .results import BccLabels


def _host_csr(g):
    off = np.ascontiguousarray(g.offsets, dtype=np.int64)
    tgt = np.asarray(g.targets)
    if tgt.dtype == np.uint32:
        tgt = tgt.view(np.int32)
    elif tgt.dtype != np.int32:
        tgt = tgt.astype(np.int32)
    return off, np.ascontiguousarray(tgt)


class _Slot:
    """A ring slot of device (or pinned host) buffers, grown on demand."""

    def __init__(self):
        self.bufs = {}

    def get(self, name, n, dtype, device, pin=False):
        t = self.bufs.get(name)
        if t is None or t.numel() < max(n, 1):
            if device == "cpu":
                t = torch.empty(max(n, 1), dtype=dtype, pin_memory=pin)
            else:
                t = torch.empty(max(n, 1), dtype=dtype, device=device)
            self.bufs[name] = t
        return t[:n]


class BccPipeline:
    """Streamed ``bcc(g)`` over an iterable of host graphs (see the module docstring)."""

    def __init__(self, device="cuda", validate=True, seed=0, trace=None):
        self.dev = torch.device(device)
        if self.dev.index is None:
            self.dev = torch.device("cuda", torch.cuda.current_device())
        self.validate = validate
        self.seed = seed
        self.trace = trace      # optional list: (graph, what, timing event) for tools/pipeline_probe.py
        self.copy_in = torch.cuda.Stream(self.dev)
        self.copy_out = torch.cuda.Stream(self.dev)
        self.compute = _priority_stream(self.dev)
        self.din = [_Slot(), _Slot()]
        self.dout = [_Slot(), _Slot()]
        self.hout = [_Slot(), _Slot()]
        self.in_free = [None, None]    # events: input slot released (BCC + symmetry check done)
        self.out_free = [None, None]   # events: output slot drained (D2H done)
        # per slot: the validation of the graph in that slot (its workspace, side stream and
        # status word) lives until that graph is finished, overlapping the next graph's
        self.vside = [torch.cuda.Stream(self.dev, priority=0), torch.cuda.Stream(self.dev, priority=0)]
        self.vslot = [_Slot(), _Slot()]

    def _mark(self, i, what, stream):
        if self.trace is not None:
            e = torch.cuda.Event(enable_timing=True)
            e.record(stream)
            self.trace.append((i, what, e))

    def _h2d(self, i, g):
        s = i % 2
        off, tgt = _host_csr(g)
        n, m = off.shape[0] - 1, tgt.shape[0]
        if n >= 2 ** 31 or m >= 2 ** 32:
            raise ValueError("graph too large for int32 vertex ids / uint32 slot ids")
        with torch.cuda.stream(self.copy_in):
            if self.in_free[s] is not None:
                self.copy_in.wait_event(self.in_free[s])
            self._mark(i, "h2d_start", self.copy_in)
            off_d = self.din[s].get("off", n + 1, torch.int64, self.dev)
            tgt_d = self.din[s].get("tgt", m, torch.int32, self.dev)
            off_d.copy_(torch.from_numpy(off), non_blocking=True)
            if m:
                tgt_d.copy_(torch.from_numpy(tgt), non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(self.copy_in)
            self._mark(i, "h2d_end", self.copy_in)
        return dict(i=i, n=n, m=m, off=off_d, tgt=tgt_d, h2d=ev)

    def _compute(self, job):
        s = job["i"] % 2
        n, m = job["n"], job["m"]
        cs = self.compute
        cs.wait_event(job["h2d"])
        with torch.cuda.stream(cs):
            self._mark(job["i"], "compute_start", cs)
            pending = None
            if self.validate:
                vws = self.vslot[s].get("ws", validate_workspace_bytes(n, m), torch.uint8, self.dev)
                pending = _validate_begin(job["off"], job["tgt"], ws=vws, side=self.vside[s])
            if self.out_free[s] is not None:
                cs.wait_event(self.out_free[s])
            lab = self.dout[s].get("lab", m, torch.int32, self.dev)
            bits = self.dout[s].get("bits", (n + 31) // 32, torch.int32, self.dev)
            cnt = self.dout[s].get("cnt", 1, torch.int64, self.dev)
            ws = _workspace(self.dev, workspace_bytes(n, m))
            lib = _lib.load()
            self._mark(job["i"], "bcc_start", cs)
            csr = _lib.PasgalCsr(n, m, job["off"].data_ptr(), job["tgt"].data_ptr() if m else 0)
            out = _lib.PasgalBccOut(lab.data_ptr() if m else 0, bits.data_ptr() if n else 0, cnt.data_ptr(), 0, 0, 0)
            st = lib.pasgal_bcc(ctypes.byref(csr), ctypes.byref(out), _vp(ws), ws.numel(),
                                int(self.seed) & (2 ** 64 - 1), 0, ctypes.c_void_p(cs.cuda_stream))
            if st != 0 and pending is not None:
                pending.finish()
            _lib.check(st, "bcc")
            art = articulation_bytes_device(bits, n)
            done = torch.cuda.Event()
            done.record(cs)
            self._mark(job["i"], "bcc_end", cs)
        # the symmetry check, queued behind the BCC kernels (it overlaps the D2H below); its
        # status word reaches pinned host memory on the same side stream
        check = None
        if pending is not None:
            vs = self.vside[s]
            vs.wait_event(done)
            # the status goes straight to pinned (mapped, under unified addressing) host memory:
            # a 4-byte D2H copy would queue behind the next graph's label copy on the copy
            # engine and hold the input slot (and so the next H2D) ~0.5 s
            st_h = self.vslot[s].get("status_h", 1, torch.int32, "cpu", pin=True)
            with torch.cuda.stream(vs):
                rc = lib.pasgal_csr_validate_check(ctypes.byref(pending.csr), _vp(pending.ws), pending.ws.numel(),
                                                   _vp(st_h), ctypes.c_void_p(vs.cuda_stream))
                _lib.check(rc, "validate")
                check = torch.cuda.Event()
                check.record(vs)
                self._mark(job["i"], "check_end", vs)
            pending.keep = None
            job.update(status_h=st_h)
        # D2H on the copy-out stream
        co = self.copy_out
        co.wait_event(done)
        with torch.cuda.stream(co):
            self._mark(job["i"], "d2h_start", co)
            hl = self.hout[s].get("lab", m, torch.int32, "cpu", pin=True)
            ha = self.hout[s].get("art", n, torch.uint8, "cpu", pin=True)
            hc = self.hout[s].get("cnt", 1, torch.int64, "cpu", pin=True)
            if m:
                hl.copy_(lab, non_blocking=True)
            if n:
                ha.copy_(art, non_blocking=True)
            hc.copy_(cnt, non_blocking=True)
            d2h = torch.cuda.Event()
            d2h.record(co)
            self._mark(job["i"], "d2h_end", co)
        self.out_free[s] = d2h
        self.in_free[s] = check if check is not None else done
        job.update(check=check, d2h=d2h, hl=hl, ha=ha, hc=hc)
        return job

    def _finish(self, job):
        if job["check"] is not None:
            job["check"].synchronize()
            _lib.check(int(job["status_h"][0]), "validate")
        job["d2h"].synchronize()
        n = job["n"]
        return BccLabels(job["ha"][:n].numpy().view(np.bool_), int(job["hc"][0]),
                         edge_label=job["hl"].numpy().view(np.uint32))

    def run(self, graphs):
        """Yield BccLabels for each graph in order.  A yielded result's arrays are views of
        pinned buffers that are overwritten once the next result is requested: copy them to
        keep them."""
        it = iter(graphs)

        def h2d(i):
            g = next(it, None)
            if g is None:
                return None
            if isinstance(g, DeviceGraph):
                raise TypeError("BccPipeline takes host graphs; use bcc_device for device-resident CSRs")
            return self._h2d(i, g)

        nxt, prev, i = h2d(0), None, 0
        while nxt is not None:
            job = self._compute(nxt)        # waits for H2D(i) + the streaming checks; queues BCC(i), D2H(i)
            nxt = h2d(i + 1)                # H2D(i+1) right away: it overlaps BCC(i) and the D2Hs
            if prev is not None:
                yield self._finish(prev)    # i-1: symmetry check status, its D2H
            prev, i = job, i + 1
        if prev is not None:
            yield self._finish(prev)
