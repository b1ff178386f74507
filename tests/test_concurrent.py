"""Concurrent FAST-BCC calls on distinct streams (the C5b batch path as bench.py times it).

include/pasgal_bcc.h promises that the library is reentrant and stream-ordered: calls on
different streams with different workspaces and outputs may overlap.  Eight C3-shaped
instances (grid 4096^2, p=0.6, seeds 2..9) run two rounds at once on four streams -- one
workspace per stream, reused by every instance dealt to it, one output per instance --
and every output of the second round is checked against the C oracle (oracle/bcc_oracle.c,
pinned to the reference by tests/test_oracle.py): canonical labels, articulation bitmap,
bcc_count.
"""

import threading

import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu

import paper_2404_17101_b200 as pg  # noqa: E402

SEEDS = list(range(2, 10))
STREAMS = 4


def _oracle_outputs(host):
    got = [None] * len(host)

    def work(i):
        off, tgt = host[i]
        r = oracle.bcc_hopcroft_tarjan(off, tgt)
        got[i] = (oracle.canonical_min_eid(off, tgt, r.edge_label), r.articulation, r.bcc_count)

    ths = [threading.Thread(target=work, args=(i,)) for i in range(len(host))]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    return got


def test_concurrent_streams_match_oracle():
    dev = torch.device("cuda", 0)
    graphs = [pg.gen_grid(4096, 4096, 0.6, s, device=dev) for s in SEEDS]
    torch.cuda.synchronize()
    nmax = max(g.n for g in graphs)
    mmax = max(g.m for g in graphs)
    streams = [torch.cuda.Stream(device=dev) for _ in range(STREAMS)]
    wss = [torch.empty(pg.workspace_bytes(nmax, mmax), dtype=torch.uint8, device=dev) for _ in range(STREAMS)]
    outs = [pg.DeviceBcc(edge_label=torch.empty(g.m, dtype=torch.int32, device=dev),
                         artic_bits=torch.empty((g.n + 31) // 32, dtype=torch.int32, device=dev),
                         bcc_count=torch.empty(1, dtype=torch.int64, device=dev)) for g in graphs]
    main = torch.cuda.current_stream(dev)
    for rnd in range(2):
        ev = torch.cuda.Event()
        ev.record(main)
        for st in streams:
            st.wait_event(ev)
        for i, g in enumerate(graphs):
            with torch.cuda.stream(streams[i % STREAMS]):
                pg.bcc_device(g.offsets, g.targets, seed=rnd * 100 + i, out=outs[i], workspace=wss[i % STREAMS])
        for st in streams:
            main.wait_stream(st)
    torch.cuda.synchronize()
    host = [(g.offsets.cpu().numpy(), g.targets.cpu().numpy().view(np.uint32)) for g in graphs]
    want = _oracle_outputs(host)
    for i, g in enumerate(graphs):
        canon = pg.canonicalize_device(g.offsets, g.targets, outs[i].edge_label, label_bound=max(g.n, 1))
        lab = canon.cpu().numpy().view(np.uint32)
        art = pg.unpack_articulation(outs[i].artic_bits.cpu().numpy(), g.n)
        cnt = int(outs[i].bcc_count.item())
        wl, wa, wc = want[i]
        assert cnt == wc, (SEEDS[i], cnt, wc)
        assert np.array_equal(art, wa), SEEDS[i]
        assert np.array_equal(lab, wl), SEEDS[i]
        # the checksum bench.py reports for each timed C5b instance agrees with the oracle's
        assert pg.canonical_checksum_device(canon, outs[i].artic_bits, outs[i].bcc_count) == \
            tuple(pg.canonical_checksum(wl, wa, wc))
