"""f4: the VGC frontier engine (csrc/vgc.cu, pasgal_bfs_vgc; SPEC.md vgc-engine and bfs).

Properties from the spec (SPEC.md run_frontier_loop / local_search / bfs_parallel):
exactness against queue BFS on directed and symmetric graphs, result invariance over
tau in {1, 4, 64, 1024}, round-count monotonicity (rounds(tau=1) >= rounds(tau=k)), the path
examples (tau = 1 -> L rounds, tau >= L -> 1 round) and the star example.  Distances are
checked against the reference's own bfs_queue outputs (tests/golden/bfs_cases.npz) and
the C oracle (oracle.bfs_queue, pinned to those goldens by tests/test_bfs.py)."""

import os

import numpy as np
import pytest

import oracle
from tests import golden_io

TAUS = (1, 4, 64, 1024)


def test_vgc_config_validation():
    import paper_2404_17101_b200 as pg

    assert pg.VgcConfig().tau == 512
    with pytest.raises(ValueError):
        pg.VgcConfig(tau=0)
    with pytest.raises(ValueError):
        pg.VgcConfig(tau=10, max_local_queue=5)
    with pytest.raises(ValueError):
        pg.VgcConfig(dense_threshold=1.5)
    assert pg.VgcConfig(dense_threshold=0.0).dense_threshold == 0.0       # always dense (tests)


def _golden_cases():
    d = np.load(os.path.join(golden_io.GOLDEN, "bfs_cases.npz"))
    oi, ti, di = d["offsets_idx"], d["targets_idx"], d["dist_idx"]
    for k, name in enumerate(d["names"]):
        off = d["offsets"][oi[k]:oi[k + 1]]
        if off.shape[0] > 1:
            yield str(name), off, d["targets"][ti[k]:ti[k + 1]], int(d["source"][k]), d["dist"][di[k]:di[k + 1]]


class _G:
    def __init__(self, off, tgt):
        self.offsets = np.ascontiguousarray(off, dtype=np.int64)
        self.targets = np.ascontiguousarray(tgt, dtype=np.uint32)


def _random_graph(rng, symmetric):
    n = int(rng.integers(1, 2000))
    m = int(rng.integers(0, 4 * n + 1))
    src = rng.integers(0, n, size=m)
    dst = rng.integers(0, n, size=m)
    if symmetric:
        src, dst = np.concatenate([src, dst]), np.concatenate([dst, src])
    order = np.lexsort((dst, src))
    src, dst = src[order], dst[order]
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(src, minlength=n), out=off[1:])
    return off, dst.astype(np.uint32)


@pytest.mark.gpu
def test_vgc_bfs_matches_reference_goldens_for_every_tau():
    import paper_2404_17101_b200 as pg

    ncase = 0
    for name, off, tgt, src, dist in _golden_cases():
        ncase += 1
        rounds = []
        for tau in TAUS:
            r = pg.bfs_parallel(_G(off, tgt), src, pg.VgcConfig(tau=tau, max_local_queue=max(tau, 2048)))
            assert np.array_equal(r.dist, dist), (name, tau)
            assert r.source == src
            rounds.append(r.rounds)
        assert rounds[0] == int(dist.max()) + 1, name          # tau = 1 is level-synchronous
        assert all(rounds[0] >= x for x in rounds[1:]), (name, rounds)
    assert ncase >= 20


@pytest.mark.gpu
def test_vgc_bfs_random_directed_and_symmetric_graphs():
    """SPEC bfs_parallel example: 200 random graphs (directed and symmetric, n <= 2000)
    equal to the queue-BFS oracle element-wise, for several tau."""
    import paper_2404_17101_b200 as pg

    rng = np.random.default_rng(2404)
    for i in range(200):
        off, tgt = _random_graph(rng, symmetric=bool(i & 1))
        n = off.shape[0] - 1
        s = int(rng.integers(0, n))
        want, _ = oracle.bfs_queue(off, tgt, s)
        tau = TAUS[i % len(TAUS)]
        got = pg.bfs_parallel(_G(off, tgt), s, pg.VgcConfig(tau=tau, max_local_queue=max(tau, 2048)))
        assert np.array_equal(got.dist, want), (i, tau)


@pytest.mark.gpu
def test_vgc_path_star_and_isolated_examples():
    import paper_2404_17101_b200 as pg

    L = 1000                                              # path 0 - 1 - ... - (L-1)
    src = np.concatenate([np.arange(1, L), np.arange(0, L - 1)])
    dst = np.concatenate([np.arange(0, L - 1), np.arange(1, L)])
    order = np.lexsort((dst, src))
    off = np.zeros(L + 1, dtype=np.int64)
    np.cumsum(np.bincount(src[order], minlength=L), out=off[1:])
    g = _G(off, dst[order])
    r1 = pg.bfs_parallel(g, 0, pg.VgcConfig(tau=1))
    assert np.array_equal(r1.dist, np.arange(L)) and r1.rounds == L
    rL = pg.bfs_parallel(g, 0, pg.VgcConfig(tau=L, max_local_queue=L))
    assert np.array_equal(rL.dist, np.arange(L)) and rL.rounds == 1
    # star: centre processed, all leaves admitted to the next frontier
    d = 5000
    off = np.concatenate([[0, d], d + np.arange(1, d + 1)]).astype(np.int64)
    tgt = np.concatenate([np.arange(1, d + 1), np.zeros(d, dtype=np.int64)])
    r = pg.bfs_parallel(_G(off, tgt), 0, pg.VgcConfig(tau=1))
    assert r.rounds == 2 and r.dist[0] == 0 and (r.dist[1:] == 1).all()
    # isolated source: one round, everything else unreachable
    off = np.array([0, 0, 1, 2], dtype=np.int64)
    tgt = np.array([2, 1], dtype=np.uint32)
    r = pg.bfs_parallel(_G(off, tgt), 0, pg.VgcConfig(tau=4))
    assert r.rounds == 1 and r.dist.tolist() == [0, -1, -1]
    with pytest.raises(ValueError):
        pg.bfs_parallel(_G(off, tgt), 3)


@pytest.mark.gpu
def test_vgc_bfs_large_diameter_grid_against_device_queue_bfs():
    """C3-sized grid (4096^2, p = 0.6): the VGC engine equals the bit-parallel BFS (itself
    pinned to the reference) for tau 1 and 1024, and the local searches cut the rounds by a
    large factor on this large-diameter graph."""
    import paper_2404_17101_b200 as pg

    dg = pg.make_config("c3")
    want = pg.bfs(dg, 0).dist
    r1 = pg.bfs_parallel(dg, 0, pg.VgcConfig(tau=1))
    rk = pg.bfs_parallel(dg, 0, pg.VgcConfig(tau=1024))
    assert np.array_equal(r1.dist, want) and np.array_equal(rk.dist, want)
    assert r1.rounds == int(want.max()) + 1
    assert rk.rounds * 4 <= r1.rounds, (r1.rounds, rk.rounds)


def _sym_random(rng, n, m):
    src = rng.integers(0, n, size=m)
    dst = rng.integers(0, n, size=m)
    keep = src != dst
    src, dst = src[keep], dst[keep]
    s2, d2 = np.concatenate([src, dst]), np.concatenate([dst, src])
    key = np.unique(s2 * n + d2)
    s2, d2 = key // n, key % n
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(s2, minlength=n), out=off[1:])
    return off, d2.astype(np.uint32)


@pytest.mark.gpu
def test_vgc_dense_rounds_equal_top_down():
    """SPEC bfs_round_dense: forced dense_threshold=0 (every round bottom-up) vs 1 (never)
    give identical DistanceArrays on 100 random symmetric graphs, for several tau; both
    equal the queue-BFS oracle."""
    import paper_2404_17101_b200 as pg

    rng = np.random.default_rng(2025)
    for i in range(100):
        n = int(rng.integers(2, 1500))
        off, tgt = _sym_random(rng, n, int(rng.integers(0, 6 * n)))
        s = int(rng.integers(0, n))
        tau = TAUS[i % len(TAUS)]
        g = _G(off, tgt)
        d0, st0 = pg.bfs_parallel(g, s, pg.VgcConfig(tau=tau, max_local_queue=max(tau, 2048), dense_threshold=0.0),
                                  symmetric=True, return_stats=True)
        d1, st1 = pg.bfs_parallel(g, s, pg.VgcConfig(tau=tau, max_local_queue=max(tau, 2048), dense_threshold=1.0),
                                  symmetric=True, return_stats=True)
        want, _ = oracle.bfs_queue(off, tgt, s)
        assert np.array_equal(d0.dist, d1.dist) and np.array_equal(d0.dist, want), (i, tau)
        assert st1["dense_rounds"] == 0
        if off[s + 1] > off[s]:                                  # threshold 0: rounds with edges go dense
            assert st0["dense_rounds"] >= 1
    # complete graph K_8 from any source: one dense round reaches everything at distance 1
    n = 8
    src = np.repeat(np.arange(n), n - 1)
    dst = np.array([w for u in range(n) for w in range(n) if w != u])
    off = np.arange(0, n * (n - 1) + 1, n - 1, dtype=np.int64)
    for s in range(n):
        d, st = pg.bfs_parallel(_G(off, dst), s, pg.VgcConfig(tau=1), symmetric=None, return_stats=True)
        assert st["dense_rounds"] >= 1 and d.dist[s] == 0 and (np.delete(d.dist, s) == 1).all()
    del src


@pytest.mark.gpu
def test_vgc_dense_rounds_on_rmat():
    """A low-diameter power-law graph (C2): with the default threshold the middle rounds go
    bottom-up; distances equal the bit-parallel BFS."""
    import paper_2404_17101_b200 as pg

    dg = pg.make_config("c2")
    want = pg.bfs(dg, 0).dist
    d, st = pg.bfs_parallel(dg, 0, pg.VgcConfig(tau=1), return_stats=True)
    assert np.array_equal(d.dist, want)
    assert st["dense_rounds"] >= 1
