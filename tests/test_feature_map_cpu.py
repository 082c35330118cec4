"""FE4D teacher-feature container (semantic.py:17-75) against a file written
by the reference's own save_feature_map (tests/golden/feature_map.feat,
make_golden.py feature_map_case): decode, byte-identical re-encode, and the
FormatError cases the reference tests (test_semantic.py:35-57).  CPU only."""

import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2503_06161_b200 import semantic as S
from paper_2503_06161_b200.errors import ConfigurationError, FormatError

PATH = os.path.join(GOLDEN, "feature_map.feat")


def test_reference_file_decodes_and_reencodes_bytes(tmp_path):
    fmap = S.load_feature_map(PATH)
    assert (fmap.channels, fmap.height, fmap.width) == (3, 5, 7)
    expect = np.random.default_rng(43).normal(size=(3, 5, 7)).astype(np.float32)
    assert np.array_equal(fmap.data, expect)
    out = tmp_path / "again.feat"
    S.save_feature_map(out, fmap)
    assert out.read_bytes() == open(PATH, "rb").read()
    assert fmap.hwc().shape == (5, 7, 3) and fmap.hwc().dtype == np.float64


def test_round_trip_bit_identical(tmp_path):
    fmap = S.FeatureMap(np.random.default_rng(1).normal(size=(16, 9, 11)).astype(np.float32))
    p1, p2 = tmp_path / "a.feat", tmp_path / "b.feat"
    S.save_feature_map(p1, fmap)
    S.save_feature_map(p2, S.load_feature_map(p1))
    assert p1.read_bytes() == p2.read_bytes()
    assert S.FeatureMap(data=fmap.data) == fmap


def test_malformed_files(tmp_path):
    blob = open(PATH, "rb").read()
    p = tmp_path / "bad.feat"
    p.write_bytes(b"NOPE" + blob[4:])
    with pytest.raises(FormatError) as ei:
        S.load_feature_map(p)
    assert ei.value.offset == 0
    p.write_bytes(blob[:10])
    with pytest.raises(FormatError) as ei:
        S.load_feature_map(p)
    assert ei.value.offset == 10
    p.write_bytes(blob[:4] + (2).to_bytes(2, "little") + blob[6:])
    with pytest.raises(FormatError, match="version") as ei:
        S.load_feature_map(p)
    assert ei.value.offset == 4
    p.write_bytes(blob[:-7])
    with pytest.raises(FormatError) as ei:
        S.load_feature_map(p)
    assert ei.value.offset == len(blob) - 7
    p.write_bytes(blob + b"\0")
    with pytest.raises(FormatError):
        S.load_feature_map(p)


def test_shape_validation():
    with pytest.raises(ConfigurationError):
        S.FeatureMap(np.zeros((4, 4)))
    with pytest.raises(ConfigurationError):
        S.FeatureMap(np.zeros((0, 4, 4)))
