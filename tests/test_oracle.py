"""CPU: pin the C oracle (oracle/bcc_oracle.c) against the reference's own outputs.

The golden fixtures were produced by the real reference (tests/golden/make_golden.py);
the restatement must reproduce them bit for bit -- raw labels (the reference's
comp_count numbering), articulation flags and bcc_count -- before it is trusted as the
parity checker at sizes the Python reference cannot reach.
"""

import os
import sys

import numpy as np
import pytest

import oracle
from tests import golden_io


@pytest.mark.parametrize("case", golden_io.all_cases(), ids=lambda c: c.name)
def test_oracle_bit_exact_vs_reference(case):
    r = oracle.bcc_hopcroft_tarjan(case.offsets, case.targets)
    assert np.array_equal(r.edge_label, case.label)
    assert np.array_equal(r.articulation, case.articulation)
    assert r.bcc_count == case.count


@pytest.mark.parametrize("case", golden_io.all_cases(), ids=lambda c: c.name)
def test_oracle_canonical_matches_reference_comparator(case):
    canon = oracle.canonical_min_eid(case.offsets, case.targets, case.label)
    assert np.array_equal(golden_io.dense_from_min_eid(case, canon), case.canon)
    # both directions of an undirected edge share the label
    src = np.repeat(np.arange(case.n), np.diff(case.offsets))
    assert np.all((canon != 0xFFFFFFFF) | (src == case.targets.astype(np.int64)))


def test_oracle_rejects_non_symmetric():
    off = np.array([0, 1, 1, 1], dtype=np.int64)
    tgt = np.array([1], dtype=np.uint32)
    with pytest.raises(ValueError, match="biconnectivity requires a symmetric graph"):
        oracle.bcc_hopcroft_tarjan(off, tgt)
    assert not oracle.is_symmetric(off, tgt)


def test_oracle_million_chain_iterative():
    """iterative oracles survive 10^6-vertex chains (no recursion)."""
    n = 1_000_000
    src = np.arange(n - 1)
    keys = np.concatenate([(src << 32) | (src + 1), ((src + 1) << 32) | src]).astype(np.uint64)
    off, tgt = oracle.csr_from_keys(n, keys)
    r = oracle.bcc_hopcroft_tarjan(off, tgt)
    assert r.bcc_count == n - 1
    assert int(r.articulation.sum()) == n - 2


def test_host_generators_pinned_to_fixtures():
    c1 = golden_io.single("c1_grid256_p06_s1.npz")
    off, tgt = oracle.gen_grid(256, 256, 0.6, 1)
    assert np.array_equal(off, c1.offsets) and np.array_equal(tgt, c1.targets)
    rm = golden_io.single("rmat_s12_d16_seed7.npz")
    off, tgt = oracle.rmat(12, 1 << 16, seed=7)
    assert np.array_equal(off, rm.offsets) and np.array_equal(tgt, rm.targets)
    kn = golden_io.single("knn_13_k5_seed3.npz")
    off, tgt = oracle.knn(1 << 13, 5, seed=3)
    assert np.array_equal(off, kn.offsets) and np.array_equal(tgt, kn.targets)


@pytest.mark.parametrize("npts,seed", [(1, 1), (5, 2), (6, 3), (100, 4), (3000, 5)])
def test_knn_cell_search_equals_brute_force(npts, seed):
    a = oracle.knn(npts, 5, seed=seed)
    b = oracle.knn(npts, 5, seed=seed, brute=True)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_grid_full_lattice_matches_reference_gen_grid():
    off, tgt = oracle.gen_grid(7, 9, 1.0, 0)
    ref = golden_io.kats()
    g10 = [c for c in ref if c.name == "grid10x10"][0]
    off10, tgt10 = oracle.gen_grid(10, 10, 1.0, 123)
    assert np.array_equal(off10, g10.offsets) and np.array_equal(tgt10, g10.targets)
    assert off[-1] == 2 * (7 * 8 + 9 * 6)


REF = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference only exists in the build container")
def test_oracle_vs_live_reference_random():
    sys.path.insert(0, REF)
    from pasgal.graph import from_edges, symmetrize
    from pasgal.oracles import bcc_hopcroft_tarjan

    rng = np.random.default_rng(99)
    for _ in range(60):
        n = int(rng.integers(1, 300))
        m = int(rng.integers(0, 3 * n + 1))
        g = symmetrize(from_edges(n, rng.integers(0, n, m), rng.integers(0, n, m)))
        ref = bcc_hopcroft_tarjan(g)
        r = oracle.bcc_hopcroft_tarjan(g.offsets, g.targets)
        assert np.array_equal(r.edge_label, ref._edge_label)
        assert np.array_equal(r.articulation, ref.articulation)
        assert r.bcc_count == ref.bcc_count


def test_oracle_connected_components_kats():
    """two disjoint triangles -> 2 components; empty n=5 -> 5."""
    kats = {c.name: c for c in golden_io.kats()}
    comp, cnt = oracle.connected_components(kats["two_triangles"].offsets, kats["two_triangles"].targets)
    assert cnt == 2 and comp.tolist() == [0, 0, 0, 3, 3, 3]
    comp, cnt = oracle.connected_components(kats["empty5"].offsets, kats["empty5"].targets)
    assert cnt == 5 and comp.tolist() == [0, 1, 2, 3, 4]
    comp, cnt = oracle.connected_components(kats["isolated_plus_edge"].offsets, kats["isolated_plus_edge"].targets)
    assert cnt == 3 and comp.tolist() == [0, 1, 1, 3]


@pytest.mark.slow
@pytest.mark.parametrize("name", ["c2", "c3", "c4"])
def test_oracle_full_size_vs_reference_hashes(name):
    """The C restatement reproduces the UNMODIFIED Python reference at full BASELINE size
    (C2 RMAT 2^20, C3 grid 4096^2, C4 kNN 2^25): raw labels (the reference's comp_count
    numbering) bit for bit, articulation, count, and the min-edge-id canonical labels.
    Hashes from tests/golden/make_fullsize_hashes.py (the reference ran 74 s / 49 s / ~10 min
    in the build container)."""
    import hashlib
    import json

    with open(os.path.join(golden_io.GOLDEN, "fullsize_ref_hashes.json")) as f:
        want = json.load(f)[name]

    def h(a):
        return hashlib.blake2b(np.ascontiguousarray(a).view(np.uint8), digest_size=16).hexdigest()

    off, tgt = {"c2": lambda: oracle.rmat(20, 1 << 24, seed=1),
                "c3": lambda: oracle.gen_grid(4096, 4096, 0.6, 1),
                "c4": lambda: oracle.knn(1 << 25, 5, seed=1)}[name]()
    assert h(off) + ":" + h(tgt) == want["csr"]
    r = oracle.bcc_hopcroft_tarjan(off, tgt)
    assert r.bcc_count == want["count"]
    assert h(r.articulation.astype(bool)) == want["artic"]
    assert h(r.edge_label.astype(np.int64)) == want["raw"]
    assert h(oracle.canonical_min_eid(off, tgt, r.edge_label)) == want["labels"]
