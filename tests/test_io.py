"""f1 graph files: header-level GraphFormatError cases need no GPU (they are raised
before any device copy); device round trips and array-level positions are GPU tests."""

import os
import struct

import numpy as np
import pytest

from tests import golden_io

pytest.importorskip("torch")
import paper_2404_17101_b200 as pg  # noqa: E402


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
