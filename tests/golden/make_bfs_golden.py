"""Generate tests/golden/bfs_cases.npz from the REAL reference (build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_bfs_golden.py

Expected values come from the reference's own code: hop distances from
``pasgal.oracles.bfs_queue`` (oracles.py:27-46) and bounds from
``pasgal.graph.estimate_diameter`` (graph.py:595-605), on graphs built with its own
``from_edges`` / ``symmetrize`` / ``gen_grid``.  Directed graphs are included: BFS and the
diameter estimate do not require symmetry.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from pasgal.graph import estimate_diameter, from_edges, gen_grid, symmetrize  # noqa: E402
from pasgal.oracles import bfs_queue  # noqa: E402


def graphs():
    rng = np.random.default_rng(77)
    out = [("path5", symmetrize(from_edges(5, np.arange(4), np.arange(1, 5)))),
           ("grid10x10", gen_grid(10, 10)),
           ("grid1x5", gen_grid(1, 5)),
           ("grid30x7", gen_grid(30, 7))]
    for i in range(24):
        n = int(rng.integers(1, 400))
        m = int(rng.integers(0, 3 * n))
        s, d = rng.integers(0, n, m), rng.integers(0, n, m)
        g = from_edges(n, s, d)
        out.append((f"rand{i}_{'sym' if i % 2 else 'dir'}", symmetrize(g) if i % 2 else g))
    # a long chain with a few shortcuts (many BFS levels)
    n = 3000
    s = np.concatenate([np.arange(n - 1), rng.integers(0, n, 5)])
    d = np.concatenate([np.arange(1, n), rng.integers(0, n, 5)])
    out.append(("chain3000", symmetrize(from_edges(n, s, d))))
    return out


def main():
    names, offs, tgts, srcs, dists, diam = [], [], [], [], [], []
    rng = np.random.default_rng(5)
    for name, g in graphs():
        names.append(name)
        offs.append(np.asarray(g.offsets, np.int64))
        tgts.append(np.asarray(g.targets, np.uint32))
        s = int(rng.integers(0, g.n)) if g.n else 0
        srcs.append(s)
        dists.append(np.asarray(bfs_queue(g, s).dist, np.int64) if g.n else np.empty(0, np.int64))
        row = []
        for samples, seed in [(1, 0), (7, 3), (100, 1), (1000, 0)]:
            row.append([samples, seed, estimate_diameter(g, samples=samples, seed=seed).diameter_lower_bound])
        diam.append(row)
    idx = lambda arrs: np.cumsum([0] + [a.shape[0] for a in arrs])  # noqa: E731
    np.savez_compressed(os.path.join(HERE, "bfs_cases.npz"), names=np.array(names),
                        offsets=np.concatenate(offs), offsets_idx=idx(offs),
                        targets=np.concatenate(tgts), targets_idx=idx(tgts),
                        source=np.array(srcs, np.int64), dist=np.concatenate(dists), dist_idx=idx(dists),
                        diameter=np.array(diam, np.int64))
    print("bfs cases", len(names))


if __name__ == "__main__":
    main()
