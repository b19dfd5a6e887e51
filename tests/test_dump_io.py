"""KVQD dumps (paper_2402_02750_b200/dump_io.py) against the reference's own
read_dump / write_dump (reference dump_io.cpp:23-105, via oracle/_ref when built):
byte-identical files, identical values, and the same FormatError byte offsets on
corrupted files (the reference's test_dump_io.cpp fixtures are byte-offset based)."""
import os
import struct

import numpy as np
import pytest

from paper_2402_02750_b200 import FormatError, ShapeError, UsageError
from paper_2402_02750_b200.dump_io import read_dump, write_dump
from oracles import Ref

HEADER = b"KVQD" + struct.pack("<IBB", 1, 0, 2) + struct.pack("<QQ", 2, 3)
PAYLOAD = np.arange(6, dtype="<f4").tobytes()

# (bytes, expected byte offset): the reference's FormatError offsets
CORRUPT = [
    (b"KVQX" + HEADER[4:] + PAYLOAD, 0),                       # bad magic
    (b"KVQD\x01\x00", 4),                                       # truncated version
    (b"KVQD" + struct.pack("<I", 2) + HEADER[8:] + PAYLOAD, 4),  # bad version
    (HEADER[:8] + b"\x01" + HEADER[9:] + PAYLOAD, 8),          # bad dtype
    (HEADER[:9] + b"\x04" + HEADER[10:] + PAYLOAD, 9),         # bad ndim
    (HEADER[:20], 18),                                          # truncated dims
    (HEADER + PAYLOAD[:10], 36),                                # truncated payload
]


@pytest.mark.parametrize("shapes", [[(3, 5)], [(4, 7)] * 3, [(1, 9)]])
def test_roundtrip(tmp_path, shapes):
    rng = np.random.default_rng(len(shapes))
    ts = [rng.standard_normal(s).astype(np.float32) for s in shapes]
    p = str(tmp_path / "a.kvqd")
    write_dump(p, ts)
    back = read_dump(p)
    assert len(back) == len(ts) and all(np.array_equal(a, b) for a, b in zip(ts, back))


def test_one_dimensional_loads_as_row(tmp_path):
    p = tmp_path / "v.kvqd"
    p.write_bytes(b"KVQD" + struct.pack("<IBB", 1, 0, 1) + struct.pack("<Q", 4) +
                  np.arange(4, dtype="<f4").tobytes())
    (m,) = read_dump(str(p))
    assert m.shape == (1, 4) and m.tolist() == [[0, 1, 2, 3]]


@pytest.mark.parametrize("blob,offset", CORRUPT)
def test_format_errors_carry_offsets(tmp_path, blob, offset):
    p = tmp_path / "bad.kvqd"
    p.write_bytes(blob)
    with pytest.raises(FormatError) as e:
        read_dump(str(p))
    assert e.value.byte_offset == offset
    if Ref.available():
        _, err = Ref().read_dump(str(p))
        assert err == (5, offset)


def test_usage_and_shape_errors(tmp_path):
    with pytest.raises(UsageError):
        write_dump(str(tmp_path / "x"), [])
    with pytest.raises(ShapeError):
        write_dump(str(tmp_path / "x"), [np.zeros((2, 2)), np.zeros((2, 3))])
    p = tmp_path / "nan.kvqd"
    write_dump(str(p), [np.array([[1.0, np.nan]], np.float32)])
    with pytest.raises(UsageError):
        read_dump(str(p))
    with pytest.raises(FormatError):
        read_dump(str(tmp_path / "missing.kvqd"))


def test_files_identical_to_reference(tmp_path):
    if not Ref.available():
        pytest.skip("oracle/_ref not built")
    ref = Ref()
    rng = np.random.default_rng(3)
    for n in (1, 4):
        ts = [rng.standard_normal((5, 8)).astype(np.float32) for _ in range(n)]
        ours, theirs = str(tmp_path / "o.kvqd"), str(tmp_path / "r.kvqd")
        write_dump(ours, ts)
        ref.write_dump(theirs, ts)
        assert open(ours, "rb").read() == open(theirs, "rb").read()
        back, err = ref.read_dump(ours)
        assert err is None and all(np.array_equal(a, b) for a, b in zip(ts, back))
