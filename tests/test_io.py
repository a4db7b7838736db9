"""SNGD binary datasets and label files (paper_2006_06743_b200.io) against the
layout the reference documents (proj/include/sng/io.hpp:28-31) and the
behaviour of proj/src/io.cpp:123-193: magic, version, header, payload, the
error types and messages, and label round trips."""
import struct

import numpy as np
import pytest

import paper_2006_06743_b200 as sng
from paper_2006_06743_b200 import io as sio


def _write_raw(path, n, dim, vals, magic=b"SNGD", version=1, cut=0):
    blob = magic + bytes([version]) + struct.pack("<QQ", n, dim) + np.asarray(vals, "<f8").tobytes()
    path.write_bytes(blob[: len(blob) - cut] if cut else blob)


def test_binary_layout_matches_reference_spec(tmp_path):
    vals = np.array([[0.1, 2.5, -3.0], [1e-300, 7.0, 1.0 / 3.0]])
    p = tmp_path / "a.sngd"
    sio.save_binary(sng.Dataset(vals), str(p))
    raw = p.read_bytes()
    assert raw[:4] == b"SNGD" and raw[4] == 1
    assert struct.unpack("<QQ", raw[5:21]) == (2, 3)
    np.testing.assert_array_equal(np.frombuffer(raw[21:], "<f8").reshape(2, 3), vals)
    ds = sio.load_binary(str(p))
    assert ds.values64 is not None  # 0.1 is not an fp32 value: the fp64 path keeps it
    np.testing.assert_array_equal(ds.values64, vals)
    assert sio.load_points(str(p)).values64 is not None


def test_fp32_exact_file_takes_fp32_path(tmp_path):
    vals = np.arange(12, dtype=np.float64).reshape(4, 3) / 4.0
    p = tmp_path / "b.sngd"
    _write_raw(p, 4, 3, vals)
    ds = sio.load_binary(str(p))
    assert ds.values64 is None and ds.values.dtype == np.float32
    np.testing.assert_array_equal(ds.values.astype(np.float64), vals)


@pytest.mark.parametrize("kind,msg", [
    ("magic", "is not an SNGD binary dataset"), ("version", "unsupported SNGD version 2"),
    ("zero", "corrupt SNGD header"), ("short", "corrupt SNGD header"),
    ("truncated", "truncated SNGD payload")])
def test_binary_errors(tmp_path, kind, msg):
    p = tmp_path / "bad.sngd"
    if kind == "magic":
        _write_raw(p, 1, 1, [1.0], magic=b"XNGD")
    elif kind == "version":
        _write_raw(p, 1, 1, [1.0], version=2)
    elif kind == "zero":
        _write_raw(p, 0, 3, [])
    elif kind == "short":
        p.write_bytes(b"SNGD\x01" + b"\x00" * 7)
    else:
        _write_raw(p, 2, 2, [1.0, 2.0, 3.0, 4.0], cut=8)
    with pytest.raises(sio.ParseError, match=msg):
        sio.load_binary(str(p))


def test_missing_file_is_io_error(tmp_path):
    with pytest.raises(sio.IoError, match="cannot open"):
        sio.load_binary(str(tmp_path / "nope.sngd"))
    with pytest.raises(sio.IoError, match="cannot open"):
        sio.load_labels(str(tmp_path / "nope.txt"))


def test_labels_round_trip_and_errors(tmp_path):
    p = tmp_path / "labels.txt"
    labels = np.array([0, 3, -1, 2, -1, 0], np.int32)
    sio.save_labels(labels, str(p))
    assert p.read_text() == "0\n3\n-1\n2\n-1\n0\n"
    np.testing.assert_array_equal(sio.load_labels(str(p)), labels)
    p.write_text("1\r\n\n-1\n")  # CRLF and blank lines are tolerated (io.cpp:182-183)
    np.testing.assert_array_equal(sio.load_labels(str(p)), [1, -1])
    p.write_text("1\n2x\n")
    with pytest.raises(sio.ParseError, match="line 2: label '2x' is not an integer"):
        sio.load_labels(str(p))
    c = sng.Clustering(labels, np.zeros(6, np.uint8), 4)
    sio.save_clustering(c, str(p))
    np.testing.assert_array_equal(sio.load_labels(str(p)), labels)
