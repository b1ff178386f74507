"""Pathological shapes: device time + parity vs the C oracle (diagnostic).

    python tools/shapes_probe.py [--scale 25]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2404_17101_b200 as pg  # noqa: E402


def shapes(scale):
    n = 1 << scale
    out = {}
    leaves = np.arange(1, n)
    out["star"] = (n, np.zeros(n - 1, np.int64), leaves)
    out["path"] = (n, np.arange(n - 1), np.arange(1, n))
    k = 3000
    a, b = np.triu_indices(k, 1)
    out["clique3000"] = (k, a, b)
    # many stars hanging off a cycle (hub heavy + long cycle)
    c = n // 1024
    cyc = np.arange(c)
    hub_s = np.repeat(cyc, 1023)
    hub_t = np.arange(c, c + c * 1023)
    out["cycle_of_stars"] = (c + c * 1023, np.concatenate([cyc, hub_s]), np.concatenate([(cyc + 1) % c, hub_t]))
    # binary tree (deep-ish, wide)
    v = np.arange(1, n)
    out["binary_tree"] = (n, (v - 1) // 2, v)
    out["matching"] = (n, np.arange(0, n, 2), np.arange(1, n, 2))
    out["selfloops_path"] = (n, np.concatenate([np.arange(n), np.arange(n - 1)]),
                             np.concatenate([np.arange(n), np.arange(1, n)]))
    out["k2n"] = (n, np.concatenate([np.zeros(n - 2, np.int64), np.ones(n - 2, np.int64)]),
                  np.concatenate([np.arange(2, n), np.arange(2, n)]))
    return out


def multi(scale):
    """one edge with multiplicity 2^(scale-3), plus a path (CSR built by hand: symmetrize
    would deduplicate)."""
    n = 1 << (scale - 3)
    k = 1 << (scale - 3)
    src = np.concatenate([np.zeros(k, np.int64), np.ones(k, np.int64), np.arange(1, n - 1), np.arange(2, n)])
    dst = np.concatenate([np.ones(k, np.int64), np.zeros(k, np.int64), np.arange(2, n), np.arange(1, n - 1)])
    order = np.lexsort((dst, src))
    src, dst = src[order], dst[order]
    off = np.concatenate([[0], np.cumsum(np.bincount(src, minlength=n))]).astype(np.int64)
    return n, off, dst.astype(np.uint32)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=25)
    ap.add_argument("--parity", action="store_true")
    a = ap.parse_args()
    items = [(k, pg.symmetrize_edges(v[0], v[1], v[2])) for k, v in shapes(a.scale).items()]
    n_m, off_m, tgt_m = multi(a.scale)
    items.append(("multiedge_path", pg.DeviceGraph(torch.from_numpy(off_m).cuda(),
                                                   torch.from_numpy(tgt_m.view(np.int32)).cuda())))
    for name, dg in items:
        n = dg.n
        pg.validate_device(dg.offsets, dg.targets)
        torch.cuda.synchronize()
        pg.bcc_device(dg.offsets, dg.targets)
        torch.cuda.synchronize()
        from paper_2404_17101_b200 import _lib

        ev = [torch.cuda.Event(enable_timing=True) for _ in _lib.STAGES]
        t0 = time.perf_counter()
        r = pg.bcc_device(dg.offsets, dg.targets, canonical=a.parity, events=ev)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) * 1e3
        st = " ".join(f"{_lib.STAGES[i]}={ev[i - 1].elapsed_time(ev[i]):.2f}" for i in range(1, len(ev)))
        line = f"{name:16s} n={n} M={dg.m} {dt:8.2f} ms bcc={int(r.bcc_count.item())} [{st}]"
        if a.parity:
            off = dg.offsets.cpu().numpy()
            tgt = dg.targets.cpu().numpy().view(np.uint32)
            ref = oracle.bcc_hopcroft_tarjan(off, tgt)
            want = oracle.canonical_min_eid(off, tgt, ref.edge_label)
            lab = r.edge_label.cpu().numpy().view(np.uint32)
            art = pg.unpack_articulation(r.artic_bits.cpu().numpy(), n)
            ok = (np.array_equal(lab, want) and np.array_equal(art, ref.articulation)
                  and int(r.bcc_count.item()) == ref.bcc_count)
            line += f" parity={'OK' if ok else 'MISMATCH'}"
        print(line, flush=True)


if __name__ == "__main__":
    main()
