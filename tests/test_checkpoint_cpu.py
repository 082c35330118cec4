"""FS4C container codec (training.py:569-674) against a file written by the
reference's own entry writer (tests/golden/checkpoint.fs4c, make_golden.py
checkpoint_case): decode, byte-identical re-encode, and the FormatError
offsets of malformed files.  CPU only."""

import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2503_06161_b200 import checkpoint as ck
from paper_2503_06161_b200.errors import FormatError

PATH = os.path.join(GOLDEN, "checkpoint.fs4c")


def test_decode_reference_file_and_reencode_bytes():
    e = ck.load_entries(PATH)
    assert e["meta.iteration"] == 7 and e["adam.positions.step"] == 3
    assert e["meta.extent"] == 1.25 and e["meta.config"] == b"[train]\nseed = 3\n"
    assert e["cloud.positions"].shape == (11, 3) and e["cloud.positions"].dtype == np.float64
    assert e["grid.l0.p2"].shape == (4, 3, 2)
    assert e["labels"].dtype == np.int64 and e["labels"].tolist() == [[0, 1, 2], [3, 4, 5]]
    with open(PATH, "rb") as fh:
        assert ck.encode_entries(e) == fh.read()


def test_round_trip(tmp_path):
    rng = np.random.default_rng(0)
    e = {"a.b": rng.normal(size=(3, 4)).astype(np.float32), "n": 5, "x": 2.5, "s": b"\x00\x01",
         "z": np.zeros((0, 3))}
    p = str(tmp_path / "c.fs4c")
    ck.write_entries(p, e)
    back = ck.load_entries(p)
    assert set(back) == set(e)
    np.testing.assert_array_equal(back["a.b"], e["a.b"])
    assert back["a.b"].dtype == np.float32 and back["z"].shape == (0, 3)
    assert back["n"] == 5 and back["x"] == 2.5 and back["s"] == b"\x00\x01"


def test_malformed_files(tmp_path):
    blob = open(PATH, "rb").read()
    p = str(tmp_path / "bad.fs4c")
    open(p, "wb").write(b"XXXX" + blob[4:])
    with pytest.raises(FormatError) as ei:
        ck.load_entries(p)
    assert ei.value.offset == 0
    open(p, "wb").write(blob[:4] + (2).to_bytes(4, "little") + blob[8:])
    with pytest.raises(FormatError, match="version"):
        ck.load_entries(p)
    open(p, "wb").write(blob[:-5])
    with pytest.raises(FormatError, match="truncated"):
        ck.load_entries(p)
