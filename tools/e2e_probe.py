"""Split one end-to-end pg.bcc(g) call into its phases (diagnostic; not a bench number).

    python tools/e2e_probe.py --config c5a

Device phases are CUDA-event timed on the current stream; host phases by perf_counter.
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2404_17101_b200 as pg  # noqa: E402

bccmod = sys.modules["paper_2404_17101_b200.bcc"]


def ev_ms(fn, reps=3):
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5a")
    a = ap.parse_args()
    dg = pg.make_config(a.config)
    n, m = dg.n, dg.m
    torch.cuda.synchronize()
    off_h = torch.empty(n + 1, dtype=torch.int64, pin_memory=True)
    tgt_h = torch.empty(m, dtype=torch.int32, pin_memory=True)
    off_h.copy_(dg.offsets)
    tgt_h.copy_(dg.targets)
    ws = bccmod._workspace(dg.offsets.device, pg.workspace_bytes(n, m))
    out = {}
    out["validate_dev_ms"] = ev_ms(lambda: pg.validate_device(dg.offsets, dg.targets, workspace=ws))
    out["bcc_dev_ms"] = ev_ms(lambda: pg.bcc_device(dg.offsets, dg.targets, workspace=ws))
    off_d = torch.empty_like(dg.offsets)
    tgt_d = torch.empty_like(dg.targets)
    out["h2d_ms"] = ev_ms(lambda: (off_d.copy_(off_h, non_blocking=True), tgt_d.copy_(tgt_h, non_blocking=True)))
    r = pg.bcc_device(dg.offsets, dg.targets, workspace=ws)
    hb = pg.HostBuffers.allocate(n, m)
    out["d2h_ms"] = ev_ms(lambda: (hb.edge_label[:m].copy_(r.edge_label, non_blocking=True),
                                   hb.articulation[:n].copy_(pg.articulation_bytes_device(r.artic_bits, n),
                                                             non_blocking=True)))
    g = pg.Graph(off_h.numpy(), tgt_h.numpy())
    pg.bcc(g, host_out=hb)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pg.bcc(g, host_out=hb)
    out["e2e_ms"] = (time.perf_counter() - t0) * 1e3
    print({k: round(v, 1) for k, v in out.items()}, "n", n, "M", m)


if __name__ == "__main__":
    main()
