"""INTEGRATION.md section 2's ctypes stub, executed verbatim.

The stub is the binding a pasgal maintainer would add (`pasgal/bcc.py`).  It is extracted
from INTEGRATION.md -- so the documented code is the tested code -- with only its relative
import of BccLabels pointed at this package's identical container (results.py:45-88), and
run on reference-shaped graphs: a `Graph` with `n`, `m`, int64 `offsets` and uint32 or
int64 `targets` (graph.py:54-129).  The dense case (M/n > 64) is the one a workspace-size
mistake breaks: validation needs 4 B per slot, FAST-BCC ~144 B per vertex.
"""

import ctypes
import os
import re

import numpy as np
import pytest

import oracle

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _stub_source():
    text = open(os.path.join(REPO, "INTEGRATION.md")).read()
    sec = text[text.index("## 2. The stub"):]
    code = re.search(r"```python\n(.*?)```", sec, re.S).group(1)
    assert "from .results import BccLabels" in code
    return code.replace("from .results import BccLabels", "from paper_2404_17101_b200.results import BccLabels")


def _load_stub():
    from paper_2404_17101_b200 import _lib

    _lib.load()
    os.environ["PASGAL_BCC_LIB"] = _lib.LIB_PATH
    ns = {"__name__": "pasgal_bcc_stub"}
    exec(compile(_stub_source(), "INTEGRATION.md#stub", "exec"), ns)
    return ns


class RefShapedGraph:
    """The reference Graph's attributes the stub reads (graph.py:54-129)."""

    def __init__(self, offsets, targets):
        self.offsets = np.asarray(offsets, dtype=np.int64)
        self.targets = targets
        self.weights = None

    @property
    def n(self):
        return self.offsets.shape[0] - 1

    @property
    def m(self):
        return int(self.targets.shape[0])


def test_stub_loads_and_binds_every_symbol_it_uses():
    """CPU: the documented module imports, loads the library and declares the sizes of
    BOTH workspaces (no device call)."""
    ns = _load_stub()
    lib = ns["_lib"]
    assert lib.pasgal_csr_validate_workspace_bytes.restype == ctypes.c_size_t
    n, m = 1 << 16, 100 << 16
    assert lib.pasgal_csr_validate_workspace_bytes(n, m) > lib.pasgal_bcc_workspace_bytes(n, m)
    assert callable(ns["bcc_parallel"])
    assert "pasgal_csr_validate_workspace_bytes(n, m)" in _stub_source()


@pytest.mark.gpu
@pytest.mark.parametrize("tdtype", [np.uint32, np.int64])
def test_stub_on_dense_rmat_matches_oracle(tdtype):
    from paper_2404_17101_b200.results import BccLabels, canonical_edge_partition

    ns = _load_stub()
    off, tgt = oracle.rmat(16, 48 << 16, seed=5)
    n, m = off.shape[0] - 1, tgt.shape[0]
    assert m / n > 64, m / n
    g = RefShapedGraph(off, tgt.astype(tdtype))
    got = ns["bcc_parallel"](g)
    ref = oracle.bcc_hopcroft_tarjan(off, tgt)
    assert got.bcc_count == ref.bcc_count
    assert np.array_equal(got.articulation, ref.articulation)
    gref = RefShapedGraph(off, tgt)
    want = canonical_edge_partition(gref, BccLabels(ref.articulation, ref.bcc_count,
                                                    edge_label=np.asarray(ref.edge_label, dtype=np.int64)))
    assert np.array_equal(canonical_edge_partition(gref, got), want)


@pytest.mark.gpu
def test_stub_raises_reference_error_on_asymmetric_graph():
    ns = _load_stub()
    g = RefShapedGraph(np.array([0, 1, 1, 1], dtype=np.int64), np.array([1], dtype=np.uint32))
    with pytest.raises(ValueError, match="biconnectivity requires a symmetric graph"):
        ns["bcc_parallel"](g)
