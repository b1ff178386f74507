"""f1 graph files: header-level GraphFormatError cases need no GPU (they are raised
before any device copy); device round trips and array-level positions are GPU tests."""

import os
import struct

import numpy as np
import pytest

from tests import golden_io

pytest.importorskip("torch")
import paper_2404_17101_b200 as pg  # noqa: E402
import torch  # noqa: E402


def _write(path, n, m, size=None, offsets=None, targets=None, extra=b""):
    size = 24 + (n + 1) * 8 + m * 4 if size is None else size
    with open(path, "wb") as f:
        f.write(struct.pack("<QQQ", n, m, size))
        if offsets is not None:
            f.write(np.asarray(offsets, dtype="<u8").tobytes())
        if targets is not None:
            f.write(np.asarray(targets, dtype="<u4").tobytes())
        f.write(extra)


def test_header_errors_are_positioned(tmp_path):
    p = tmp_path / "a.bin"
    p.write_bytes(b"\x00" * 10)
    with pytest.raises(pg.GraphFormatError, match=r"truncated file: 10 bytes.*byte 10"):
        pg.load_bin(p)
    _write(p, 2, 2, size=7, offsets=[0, 1, 2], targets=[1, 0])
    with pytest.raises(pg.GraphFormatError, match=r"size-field mismatch.*byte 16") as e:
        pg.load_bin(p)
    assert isinstance(e.value, ValueError) and e.value.byte == 16
    _write(p, 2, 2, offsets=[0, 1, 2], targets=[1])
    with pytest.raises(pg.GraphFormatError, match="truncated file"):
        pg.load_bin(p)
    _write(p, 2, 2, offsets=[1, 1, 2], targets=[1, 0])
    with pytest.raises(pg.GraphFormatError, match=r"offset block invalid.*byte 24"):
        pg.load_bin(p)
    _write(p, 2 ** 31, 0)
    with pytest.raises(pg.GraphFormatError, match="exceeds"):
        pg.load_bin(p)


def test_reference_written_file_header_is_accepted():
    """The fixture was written by pasgal.graph.save_bin; its header parses like ours."""
    path = os.path.join(golden_io.GOLDEN, "grid10x10_ref.bin")
    data = open(path, "rb").read()
    n, m, size = struct.unpack_from("<QQQ", data, 0)
    assert (n, m, size) == (100, 360, 24 + 101 * 8 + 360 * 4) == (n, m, len(data))


@pytest.mark.gpu
def test_device_load_bin_round_trip_and_positions(tmp_path):
    kat = [c for c in golden_io.kats() if c.name == "grid10x10"][0]
    g = pg.load_bin(os.path.join(golden_io.GOLDEN, "grid10x10_ref.bin"))
    assert np.array_equal(g.offsets.cpu().numpy(), kat.offsets)
    assert np.array_equal(g.targets.cpu().numpy().view(np.uint32), kat.targets)
    r = pg.bcc(g)
    assert r.bcc_count == kat.count and np.array_equal(r.articulation, kat.articulation)
    # our writer round-trips a BASELINE graph
    dg = pg.make_config("c2")
    p = tmp_path / "c2.bin"
    pg.save_bin(dg, p)
    g2 = pg.load_bin(p)
    assert np.array_equal(g2.offsets.cpu().numpy(), dg.offsets.cpu().numpy())
    assert np.array_equal(g2.targets.cpu().numpy(), dg.targets.cpu().numpy())
    # array-level errors carry the reference's byte positions
    _write(p, 3, 2, offsets=[0, 2, 1, 2], targets=[1, 0])
    with pytest.raises(pg.GraphFormatError, match=r"offsets decrease at index 2.*byte 40"):
        pg.load_bin(p)
    _write(p, 3, 2, offsets=[0, 1, 2, 2], targets=[1, 7])
    with pytest.raises(pg.GraphFormatError, match=r"target out of range at edge 1: 7 >= n=3.*byte 60"):
        pg.load_bin(p)


# ---------------------------------------------------------------------------------------
# text adjacency files (load_adj / save_adj, graph.py:250-336)
# ---------------------------------------------------------------------------------------

def _adj_cases():
    import base64
    import json

    with open(os.path.join(golden_io.GOLDEN, "adj_cases.json")) as f:
        cases = json.load(f)
    for c in cases:
        c["data"] = base64.b64decode(c["data_b64"])
    return cases


def test_adj_fixture_covers_every_reference_check():
    """The reference-generated cases (tests/golden/make_adj_golden.py) exercise every
    message load_adj can raise, the OverflowError path, and successful loads."""
    cases = _adj_cases()
    msgs = {c["expect"].get("message", "ok").split(" (")[0].split(" at ")[0].split(":")[0].split(" b'")[0]
            for c in cases}
    for want in ["empty file, missing header", "malformed header", "missing vertex/edge counts",
                 "invalid count token", "negative counts n=-1 m=0", "token count mismatch",
                 "invalid offset token", "first offset must be 0", "offset out of range",
                 "invalid target token", "target out of range", "invalid weight token",
                 "negative or invalid weight", "Python int too large to convert to C long", "ok"]:
        assert any(m.startswith(want) for m in msgs), want
    assert len(cases) >= 200


def test_save_adj_matches_reference_bytes(tmp_path):
    """Our writer produces the reference's canonical serialization byte for byte."""
    kat = [c for c in golden_io.kats() if c.name == "grid10x10"][0]
    p = tmp_path / "g.adj"
    pg.save_adj(pg.Graph(kat.offsets, kat.targets), p)
    assert p.read_bytes() == open(os.path.join(golden_io.GOLDEN, "grid10x10_ref.adj"), "rb").read()


@pytest.mark.gpu
def test_device_load_adj_matches_reference_on_every_case(tmp_path):
    for c in _adj_cases():
        p = tmp_path / "case.adj"
        p.write_bytes(c["data"])
        e = c["expect"]
        if "error" in e:
            with pytest.raises(Exception) as ex:
                pg.load_adj(p, c["weighted"])
            assert type(ex.value).__name__ == e["error"], c["name"]
            assert str(ex.value) == e["message"].replace("{path}", str(p)), c["name"]
        else:
            g = pg.load_adj(p, c["weighted"])
            assert g.n == e["n"] and g.m == e["m"], c["name"]
            assert g.offsets.cpu().numpy().tolist() == e["offsets"], c["name"]
            assert g.targets.cpu().numpy().tolist() == e["targets"], c["name"]


@pytest.mark.gpu
def test_device_load_adj_reference_file_and_round_trip(tmp_path):
    kat = [c for c in golden_io.kats() if c.name == "grid10x10"][0]
    g = pg.load_adj(os.path.join(golden_io.GOLDEN, "grid10x10_ref.adj"))
    assert np.array_equal(g.offsets.cpu().numpy(), kat.offsets)
    assert np.array_equal(g.targets.cpu().numpy().view(np.uint32), kat.targets)
    r = pg.bcc(g)
    assert r.bcc_count == kat.count and np.array_equal(r.articulation, kat.articulation)
    # multi-tile file: a BASELINE graph through save_adj -> device parse
    dg = pg.gen_rmat(16, 1 << 20, seed=3)
    p = tmp_path / "rmat16.adj"
    pg.save_adj(dg, p)
    assert p.stat().st_size > 4 * 4096
    g2 = pg.load_adj(p)
    assert torch.equal(g2.offsets, dg.offsets) and torch.equal(g2.targets, dg.targets)


# ---------------------------------------------------------------------------------------
# load_graph dispatch and the .wbin weight block (graph.py:384-390, 411-418)
# ---------------------------------------------------------------------------------------

def _bin_cases():
    import base64
    import json

    with open(os.path.join(golden_io.GOLDEN, "bin_cases.json")) as f:
        cases = json.load(f)
    for c in cases:
        c["data"] = base64.b64decode(c["data_b64"])
    return cases


def _check_case(c, p, load):
    e = c["expect"]
    if "error" in e:
        with pytest.raises(Exception) as ex:
            load(p)
        assert type(ex.value).__name__ == e["error"], c["name"]
        assert str(ex.value) == e["message"].replace("{path}", str(p)), c["name"]
    else:
        g = load(p)
        assert g.n == e["n"] and g.m == e["m"], c["name"]
        assert g.offsets.cpu().numpy().tolist() == e["offsets"], c["name"]
        assert g.targets.cpu().numpy().view(np.uint32).tolist() == e["targets"], c["name"]


def test_load_graph_host_level_cases(tmp_path):
    """Cases the reference rejects before touching arrays (extension dispatch, truncated
    weight block) raise the same error, at the same position, with no device work."""
    host = [c for c in _bin_cases() if "unknown graph extension" in c["expect"].get("message", "")
            or "truncated" in c["expect"].get("message", "")]
    assert len(host) >= 4
    for c in host:
        p = tmp_path / c["name"]
        p.write_bytes(c["data"])
        _check_case(c, p, pg.load_graph)


def test_load_bin_rejects_slot_count_beyond_uint32(tmp_path):
    p = tmp_path / "big.bin"
    _write(p, 2, 2 ** 32)
    with pytest.raises(pg.GraphFormatError, match=r"edge count 4294967296 exceeds.*byte 8"):
        pg.load_bin(p)


@pytest.mark.gpu
def test_device_load_graph_matches_reference_on_every_case(tmp_path):
    """Every reference-generated case (tests/golden/make_bin_golden.py): negative weights
    positioned at the first offender, NaN / -0.0 accepted like weights.min() < 0, .adj and
    .bin dispatch, unknown extensions."""
    for c in _bin_cases():
        p = tmp_path / c["name"]
        p.write_bytes(c["data"])
        _check_case(c, p, pg.load_graph)
