"""CPU: the host side of the drop-in -- the C-ABI library loads and exports every symbol
the header declares, argument errors map to the reference's exceptions, the workspace
is O(n), the results mirror reproduces the reference comparator, and the product never
touches the oracle.  No compute call is made (there is no GPU here)."""

import ctypes
import os
import re

import numpy as np
import pytest

from tests import golden_io

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "pasgal_bcc.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2404_17101_b200 import _build, _lib

    _build.build()
    return _lib.load()


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pasgal_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_expected_entry_points():
    fns = header_functions()
    for f in ["pasgal_bcc", "pasgal_bcc_workspace_bytes", "pasgal_csr_validate", "pasgal_strerror",
              "pasgal_csr_from_keys", "pasgal_gen_grid", "pasgal_gen_rmat_keys", "pasgal_gen_knn_keys"]:
        assert f in fns


def test_library_exports_every_declared_symbol(lib):
    from paper_2404_17101_b200 import _lib

    for name in header_functions():
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} has no ctypes signature"


def test_strerror_and_version(lib):
    from paper_2404_17101_b200 import _lib

    assert _lib.strerror(2) == "biconnectivity requires a symmetric graph"
    assert b"sm_100a" in lib.pasgal_version()
    for code in range(0, 8):
        assert isinstance(_lib.strerror(code), str)


def test_status_mapping_to_reference_exceptions():
    from paper_2404_17101_b200 import _lib

    _lib.check(0)
    with pytest.raises(ValueError, match="^biconnectivity requires a symmetric graph$"):
        _lib.check(_lib.PASGAL_ENOTSYM)
    for code in (_lib.PASGAL_EINVAL, _lib.PASGAL_EWORKSPACE, _lib.PASGAL_EUNSORTED, _lib.PASGAL_ERANGE):
        with pytest.raises(ValueError):
            _lib.check(code)
    with pytest.raises(_lib.PasgalError):
        _lib.check(_lib.PASGAL_ECUDA)


def test_argument_checks_need_no_gpu(lib):
    """Invalid arguments are rejected on the host before any CUDA call."""
    from paper_2404_17101_b200 import _lib

    out = _lib.PasgalBccOut(0, 0, 0, 0, 0, 0)
    assert lib.pasgal_bcc(None, ctypes.byref(out), None, 0, 0, 0, None) == _lib.PASGAL_EINVAL
    bad = _lib.PasgalCsr(-1, 0, 1, 0)
    assert lib.pasgal_bcc(ctypes.byref(bad), ctypes.byref(out), None, 0, 0, 0, None) == _lib.PASGAL_EINVAL
    big = _lib.PasgalCsr(1 << 31, 0, 1, 0)
    assert lib.pasgal_bcc(ctypes.byref(big), ctypes.byref(out), None, 0, 0, 0, None) == _lib.PASGAL_EINVAL
    ok = _lib.PasgalCsr(4, 0, 1, 0)
    # missing outputs
    assert lib.pasgal_bcc(ctypes.byref(ok), ctypes.byref(out), None, 0, 0, 0, None) == _lib.PASGAL_EINVAL
    out2 = _lib.PasgalBccOut(0, 8, 8, 0, 0, 0)
    assert lib.pasgal_bcc(ctypes.byref(ok), ctypes.byref(out2), None, 0, 0, 0, None) == _lib.PASGAL_EWORKSPACE
    assert lib.pasgal_gen_rmat_keys(10, 10, 1, 5, 4, 3, 8, 8, None) == _lib.PASGAL_EINVAL


def test_workspace_is_linear_in_n(lib):
    """auxiliary space O(n); the only M-dependent parts are the warp-chunk
    row partition (4 bytes per 256 slots) and the scan status (8 bytes per 2048 items)."""
    for n in [1, 1000, 1 << 20, 1 << 28]:
        base = lib.pasgal_bcc_workspace_bytes(n, 0)
        assert base <= 200 * n + (1 << 20)
        m = 50 * n
        extra = lib.pasgal_bcc_workspace_bytes(n, m) - base
        assert extra <= 4 * (m // 256 + 2) + 8 * (m // 2048 + 2) + 4096


def test_workspace_non_decreasing_in_n(lib):
    """the list-ranking ruler spacing coarsens with n (2^18, 2^25, 2^28), so the
    ruler arrays are sized for the largest count any smaller graph needs -- a workspace
    sized for the largest graph of a batch must fit every smaller one."""
    prev = 0
    pts = []
    for t in (1 << 18, 1 << 25, 1 << 28):
        pts += [t - 2, t - 1, t, t + 1]
    pts += [1, 2, 1000, (1 << 20) + 3, (1 << 30)]
    for n in sorted(pts):
        b = lib.pasgal_bcc_workspace_bytes(n, 0)
        assert b >= prev, n
        prev = b


def test_validate_workspace_is_linear_in_m(lib):
    """Validation scratch: one 8-byte key per run of up slots (<= m/2) plus per-CTA
    histograms; an undersized workspace is refused before any device work."""
    for n, m in [(1, 0), (1000, 10), (1 << 20, 50 << 20), (1 << 28, 16 << 28)]:
        need = lib.pasgal_csr_validate_workspace_bytes(n, m)
        assert 4 * m <= need <= 4 * m + m // 64 + 2 * 4096 * 1184 + (1 << 20)
    from paper_2404_17101_b200 import _lib

    csr = _lib.PasgalCsr(10, 20, 0x1000, 0x2000)
    need = lib.pasgal_csr_validate_workspace_bytes(10, 20)
    assert lib.pasgal_csr_validate(ctypes.byref(csr), ctypes.c_void_p(0x3000), need - 1, None) == _lib.PASGAL_EWORKSPACE


def test_results_mirror_matches_reference_comparator():
    from paper_2404_17101_b200.results import BccLabels, canonical_edge_partition, canonical_relabel

    for case in golden_io.all_cases():
        b = BccLabels(case.articulation, case.count, edge_label=case.label.astype(np.int64))
        assert np.array_equal(canonical_edge_partition(case, b), case.canon), case.name
    assert canonical_relabel(np.array([7, 7, 3, 9, 3])).tolist() == [0, 0, 1, 2, 1]
    assert canonical_relabel(np.array([], dtype=np.int64)).shape == (0,)


def test_min_eid_labels_give_reference_partition():
    import oracle
    from paper_2404_17101_b200.results import min_eid_to_partition

    for case in golden_io.kats() + golden_io.corpus()[:50]:
        canon = oracle.canonical_min_eid(case.offsets, case.targets, case.label)
        assert np.array_equal(min_eid_to_partition(case, canon), case.canon)


def test_uint32_labels_decode_unlabelled_as_minus_one():
    from paper_2404_17101_b200.results import BccLabels

    b = BccLabels(np.zeros(2, bool), 0, edge_label=np.array([0xFFFFFFFF, 5], dtype=np.uint32))
    assert b.edge_labels(None).tolist() == [-1, 5]


def test_product_never_imports_oracle():
    pkg = os.path.join(REPO, "paper_2404_17101_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(root, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", src, re.M), f
                assert "liboracle" not in src, f


def test_unpack_articulation_bit_order():
    from paper_2404_17101_b200.bcc import unpack_articulation

    bits = np.array([0b101, 1 << 31, 1], dtype=np.uint32)
    a = unpack_articulation(bits, 70)
    assert np.flatnonzero(a).tolist() == [0, 2, 63, 64]


def test_generator_thresholds_match_oracle_twin():
    import oracle
    from paper_2404_17101_b200.graph import grid_threshold, knn_gbits, rmat_thresholds

    for p in [0.0, 0.1, 0.5, 0.6, 0.999, 1.0]:
        assert grid_threshold(p) == oracle.grid_threshold(p)
    assert rmat_thresholds(0.57, 0.19, 0.19) == oracle.rmat_thresholds(0.57, 0.19, 0.19)
    for n in [1, 7, 100, 1 << 20, 1 << 25]:
        assert knn_gbits(n) == oracle.knn_gbits(n)


def test_canonical_checksum_rule():
    from paper_2404_17101_b200.results import canonical_checksum

    lab = np.array([0, 0, 2, 0xFFFFFFFF, 2], dtype=np.uint32)
    art = np.array([False, True, True])
    c, a, h = canonical_checksum(lab, art, 2)
    assert (c, a) == (2, 2)
    w = [((s * 0x9E3779B1) % (1 << 32)) | 1 for s in range(5)]
    assert h == sum(int(x) * y for x, y in zip(lab, w)) % (1 << 64)
    assert canonical_checksum(lab[::-1].copy(), art, 2)[2] != h      # slot order matters
