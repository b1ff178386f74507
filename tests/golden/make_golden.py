"""Generate tests/golden/*.npz from the REAL reference (run in the build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every expected output below is produced by the reference's own code --
pasgal.oracles.bcc_hopcroft_tarjan (oracles.py:119-201) and
pasgal.results.canonical_edge_partition (results.py:103-112) -- on graphs built with the
reference's own builders (from_edges / symmetrize / gen_grid, graph.py:176-194, 452-508)
or, for the BASELINE-shaped cases the reference cannot generate (grid with keep
probability, RMAT, kNN), with this repo's host generator twins (oracle/gen_host.c).
/root/reference does not exist on the GPU box, so the fixtures are committed.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

from pasgal.graph import Graph, from_edges, gen_grid, save_bin, symmetrize  # noqa: E402
from pasgal.oracles import bcc_hopcroft_tarjan  # noqa: E402
from pasgal.results import canonical_edge_partition  # noqa: E402

import oracle  # noqa: E402  (host generator twins only)


def ref_case(g):
    r = bcc_hopcroft_tarjan(g)
    return dict(
        offsets=np.asarray(g.offsets, dtype=np.int64),
        targets=np.asarray(g.targets, dtype=np.uint32),
        label=np.asarray(r._edge_label, dtype=np.int32),
        artic=np.packbits(np.asarray(r.articulation, dtype=np.uint8), bitorder="little"),
        count=np.int64(r.bcc_count),
        canon=np.asarray(canonical_edge_partition(g, r), dtype=np.int32),
    )


def sym(n, edges):
    e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    return symmetrize(from_edges(n, e[:, 0], e[:, 1]))


def kats():
    """SPEC.md:417-420, 442-445 known-answer graphs (+ a few more shapes)."""
    cases = {
        "triangle": sym(3, [(0, 1), (1, 2), (2, 0)]),
        "path3": sym(3, [(0, 1), (1, 2)]),
        "two_triangles": sym(6, [(0, 1), (1, 2), (2, 0), (3, 4), (4, 5), (5, 3)]),
        "empty5": Graph(np.zeros(6, dtype=np.int64), np.empty(0, dtype=np.uint32)),
        "star4": sym(5, [(0, 1), (0, 2), (0, 3), (0, 4)]),
        "bowtie": sym(5, [(0, 1), (1, 2), (2, 0), (2, 3), (3, 4), (4, 2)]),
        "k4": sym(4, [(a, b) for a in range(4) for b in range(a + 1, 4)]),
        "isolated_plus_edge": sym(4, [(1, 2)]),
        "chain1000": sym(1000, [(i, i + 1) for i in range(999)]),
        "cycle1000": sym(1000, [(i, (i + 1) % 1000) for i in range(1000)]),
        "two_triangles_on_nonroot": sym(7, [(0, 1), (1, 2), (2, 3), (3, 1), (2, 4), (4, 5), (5, 2), (0, 6)]),
        "grid10x10": gen_grid(10, 10),
        "single_vertex": Graph(np.zeros(2, dtype=np.int64), np.empty(0, dtype=np.uint32)),
        "zero_vertices": Graph(np.zeros(1, dtype=np.int64), np.empty(0, dtype=np.uint32)),
        # multigraph + self-loop: the reference pairs parallel edges by twin and leaves
        # self-loop slots unlabelled (-1)
        "multi_edge": Graph(*_multi()),
        # vertex 1's only slot is a self-loop: it is isolated in the spanning forest
        "selfloop_only": Graph(np.array([0, 1, 2, 3], dtype=np.int64), np.array([2, 1, 0], dtype=np.uint32)),
    }
    return cases


def _multi():
    # 0-1 double edge, 1-2 single edge, self-loop at 2, triangle 2-3-4
    adj = {0: [1, 1], 1: [0, 0, 2], 2: [1, 2, 3, 4], 3: [2, 4], 4: [2, 3]}
    off = [0]
    tgt = []
    for v in range(5):
        tgt += adj[v]
        off.append(len(tgt))
    return np.array(off, dtype=np.int64), np.array(tgt, dtype=np.uint32)


def corpus(seed=20240426):
    """Random corpus in the shape of SPEC.md:626 (ER densities, grids, chains, stars,
    cliques, cactus-like), all symmetrised by the reference's symmetrize."""
    rng = np.random.default_rng(seed)
    out = []
    for i in range(240):
        kind = i % 6
        if kind <= 2:
            n = int(rng.integers(1, 400))
            dens = [0.5, 1, 2, 8][int(rng.integers(0, 4))]
            m = int(n * dens)
            g = symmetrize(from_edges(n, rng.integers(0, n, m), rng.integers(0, n, m)))
        elif kind == 3:
            r, c = int(rng.integers(1, 40)), int(rng.integers(1, 40))
            full = gen_grid(r, c)
            src = np.repeat(np.arange(full.n), np.diff(full.offsets))
            dst = full.targets.astype(np.int64)
            keep = (src < dst) & (rng.random(src.shape[0]) < 0.6)
            g = symmetrize(from_edges(full.n, src[keep], dst[keep]))
        elif kind == 4:
            n = int(rng.integers(2, 500))
            par = [int(rng.integers(max(0, v - 4), v)) for v in range(1, n)]
            extra = int(rng.integers(0, n // 3 + 1))
            s = np.concatenate([np.arange(1, n), rng.integers(0, n, extra)])
            d = np.concatenate([np.array(par, dtype=np.int64), rng.integers(0, n, extra)])
            g = symmetrize(from_edges(n, s, d))
        else:
            # stars + cliques glued at random vertices
            n = int(rng.integers(5, 200))
            edges = []
            hub = int(rng.integers(0, n))
            for v in range(n):
                if v != hub and rng.random() < 0.3:
                    edges.append((hub, v))
            for _ in range(int(rng.integers(1, 4))):
                k = int(rng.integers(3, 8))
                vs = rng.choice(n, size=min(k, n), replace=False)
                edges += [(int(a), int(b)) for a in vs for b in vs if a < b]
            g = sym(n, edges) if edges else Graph(np.zeros(n + 1, dtype=np.int64), np.empty(0, np.uint32))
        out.append(g)
    return out


def pack_cases(cases):
    """Concatenate many small cases into flat arrays + index arrays."""
    keys = ["offsets", "targets", "label", "artic", "canon"]
    flat = {k: [] for k in keys}
    idx = {k: [0] for k in keys}
    counts = []
    for c in cases:
        for k in keys:
            flat[k].append(c[k])
            idx[k].append(idx[k][-1] + c[k].shape[0])
        counts.append(c["count"])
    res = {k: np.concatenate(flat[k]) if flat[k] else np.empty(0) for k in keys}
    for k in keys:
        res[k + "_idx"] = np.array(idx[k], dtype=np.int64)
    res["count"] = np.array(counts, dtype=np.int64)
    return res


def main():
    os.makedirs(HERE, exist_ok=True)
    kat = kats()
    names = list(kat.keys())
    cases = [ref_case(kat[k]) for k in names]
    np.savez_compressed(os.path.join(HERE, "kats.npz"), names=np.array(names), **pack_cases(cases))
    print("kats", len(cases))

    corp = [ref_case(g) for g in corpus()]
    np.savez_compressed(os.path.join(HERE, "corpus.npz"), **pack_cases(corp))
    print("corpus", len(corp), "graphs, slots", sum(c["targets"].shape[0] for c in corp))

    # a binary graph file written by the reference's own save_bin (graph.py:398-409): the
    # device loader must read it back identically
    save_bin(kat["grid10x10"], os.path.join(HERE, "grid10x10_ref.bin"))
    print("grid10x10_ref.bin written by pasgal.graph.save_bin")

    # BASELINE configs[0] (C1): grid 256x256, p=0.6, seed 1 -- CSR from the host twin of
    # the device generator, expected outputs from the reference oracle
    off, tgt = oracle.gen_grid(256, 256, 0.6, 1)
    c1 = ref_case(Graph(off, tgt))
    np.savez_compressed(os.path.join(HERE, "c1_grid256_p06_s1.npz"), **c1)
    print("c1", c1["targets"].shape[0], "slots, bcc", int(c1["count"]))

    # small RMAT / kNN in the BASELINE shapes (generator twins + reference oracle)
    off, tgt = oracle.rmat(12, 1 << 16, seed=7)
    r = ref_case(Graph(off, tgt))
    np.savez_compressed(os.path.join(HERE, "rmat_s12_d16_seed7.npz"), **r)
    print("rmat12", r["targets"].shape[0], "slots, bcc", int(r["count"]))
    off, tgt = oracle.knn(1 << 13, 5, seed=3)
    r = ref_case(Graph(off, tgt))
    np.savez_compressed(os.path.join(HERE, "knn_13_k5_seed3.npz"), **r)
    print("knn13", r["targets"].shape[0], "slots, bcc", int(r["count"]))


if __name__ == "__main__":
    main()
