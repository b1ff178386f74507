"""f4: BFS hop distances and sampled diameter estimation.

The C oracle (oracle.bfs_queue / oracle.estimate_diameter) is pinned to the reference's own
bfs_queue and estimate_diameter outputs (tests/golden/bfs_cases.npz, made by
tests/golden/make_bfs_golden.py); the device engine (csrc/bfs.cu, 64 sources per pass) is
checked against both."""

import os

import numpy as np
import pytest

import oracle
from tests import golden_io

GOLDEN = os.path.join(golden_io.GOLDEN, "bfs_cases.npz")


def _cases():
    d = np.load(GOLDEN)
    oi, ti, di = d["offsets_idx"], d["targets_idx"], d["dist_idx"]
    for k, name in enumerate(d["names"]):
        yield (str(name), d["offsets"][oi[k]:oi[k + 1]], d["targets"][ti[k]:ti[k + 1]], int(d["source"][k]),
               d["dist"][di[k]:di[k + 1]], d["diameter"][k])


def test_oracle_bfs_and_diameter_match_reference():
    n_cases = 0
    for name, off, tgt, src, dist, diam in _cases():
        n_cases += 1
        if off.shape[0] > 1:
            got, ecc = oracle.bfs_queue(off, tgt, src)
            assert np.array_equal(got, dist), name
            assert ecc == int(dist.max()), name
        for samples, seed, want in diam:
            assert oracle.estimate_diameter(off, tgt, int(samples), int(seed)) == want, name
    assert n_cases >= 25


def test_oracle_bfs_rejects_bad_source():
    with pytest.raises(ValueError, match="source 3 out of range for n=3"):
        oracle.bfs_queue(np.array([0, 0, 0, 0]), np.empty(0, np.uint32), 3)


torch = pytest.importorskip("torch")
import paper_2404_17101_b200 as pg  # noqa: E402


@pytest.mark.gpu
def test_device_bfs_and_diameter_match_reference():
    for name, off, tgt, src, dist, diam in _cases():
        g = pg.Graph(off, tgt)
        if g.n:
            r = pg.bfs(g, src)
            assert np.array_equal(r.dist, dist), name
            assert r.source == src and r.rounds == int(dist.max()), name
        for samples, seed, want in diam:
            s = pg.estimate_diameter(g, samples=int(samples), seed=int(seed))
            assert (s.n, s.m, s.diameter_lower_bound, s.sample_count) == (g.n, g.m, int(want), int(samples)), name


@pytest.mark.gpu
def test_device_eccentricities_batches_match_oracle():
    """64-source passes (with repeated sources) on BASELINE-shaped graphs and a long path."""
    rng = np.random.default_rng(9)
    graphs = [pg.make_config("c1"), pg.gen_rmat(14, 1 << 18, seed=2), pg.gen_knn(1 << 13, 5, seed=4)]
    n = 20000
    src = np.arange(n - 1)
    graphs.append(pg.symmetrize_edges(n, src, src + 1))
    for dg in graphs:
        off = dg.offsets.cpu().numpy()
        tgt = dg.targets.cpu().numpy().view(np.uint32)
        sources = rng.integers(0, dg.n, 70).tolist()
        sources[5] = sources[3]
        got = pg.eccentricities(dg, sources)
        want = [oracle.bfs_queue(off, tgt, s)[1] for s in sources]
        assert got == want
        d = pg.bfs(dg, sources[0])
        assert np.array_equal(d.dist, oracle.bfs_queue(off, tgt, sources[0])[0])


@pytest.mark.gpu
def test_bounded_diameter_equals_unbounded():
    """Skipping bounded samples never changes the estimate (symmetric graphs)."""
    graphs = [pg.make_config("c1"), pg.gen_knn(1 << 14, 5, seed=8), pg.gen_grid(300, 200, 0.7, 5),
              pg.gen_rmat(13, 1 << 16, seed=4)]
    for dg in graphs:
        for samples, seed in [(100, 0), (1000, 3)]:
            a = pg.estimate_diameter(dg, samples=samples, seed=seed, bound=True)
            b = pg.estimate_diameter(dg, samples=samples, seed=seed, bound=False)
            assert a == b
    off = graphs[0].offsets.cpu().numpy()
    tgt = graphs[0].targets.cpu().numpy().view(np.uint32)
    assert pg.estimate_diameter(graphs[0], 300, 1).diameter_lower_bound == oracle.estimate_diameter(off, tgt, 300, 1)


@pytest.mark.gpu
def test_device_bfs_directed_and_errors():
    # directed chain 0 -> 1 -> 2, 3 isolated
    g = pg.Graph(np.array([0, 1, 2, 2, 2]), np.array([1, 2], np.uint32))
    assert pg.bfs(g, 0).dist.tolist() == [0, 1, 2, -1]
    assert pg.bfs(g, 2).dist.tolist() == [-1, -1, 0, -1]
    with pytest.raises(ValueError, match="source 4 out of range for n=4"):
        pg.bfs(g, 4)
    with pytest.raises(ValueError, match="samples must be >= 1"):
        pg.estimate_diameter(g, samples=0)
    assert pg.estimate_diameter(pg.Graph(np.zeros(4, np.int64), np.empty(0, np.uint32))).diameter_lower_bound == 0
