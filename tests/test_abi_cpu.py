"""CPU-side checks of the C-ABI boundary: the in-tree library loads, exports
every symbol include/fs4d.h declares, and the ctypes layouts match the header
(no compute calls: there is no GPU here)."""

import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "fs4d.h")


def _declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(fs4d_\w+)\s*\(", txt, re.M)))


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__ as ge
    ge.build()
    from paper_2503_06161_b200 import _native
    return _native.load()


def test_header_declares_entry_points():
    names = _declared()
    for must in ("fs4d_render_fwd", "fs4d_render_bwd", "fs4d_deform_fwd", "fs4d_deform_bwd",
                 "fs4d_render_workspace_bytes", "fs4d_deform_workspace_bytes", "fs4d_status_reset"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    for name in _declared():
        assert hasattr(lib, name), name


def test_ctypes_signatures_cover_header(lib):
    from paper_2503_06161_b200 import _native
    assert set(_declared()) == set(_native.SIGNATURES)


def test_abi_version_and_build_info(lib):
    assert lib.fs4d_abi_version() == 1
    assert b"sm_100a" in lib.fs4d_build_info()


def test_struct_sizes_match_header_layout():
    from paper_2503_06161_b200 import _native as N
    # int64 + 2*int32 + 7 pointers
    assert ctypes.sizeof(N.Cloud) == 8 + 8 + 7 * 8
    assert ctypes.sizeof(N.Camera) == 8 + 9 * 8 + 16 * 8
    assert ctypes.sizeof(N.RecordInfo) == 8 + 6 * 4 + 8
    assert ctypes.sizeof(N.Linear) == 8 + 8 + 3 * 4 + 4  # padded to 8


def test_workspace_sizing_is_host_only(lib):
    from paper_2503_06161_b200 import _native as N
    info = N.RecordInfo()
    info.K, info.height, info.width, info.D, info.tile, info.pair_capacity = 200000, 512, 640, 16, 16, 2000000
    nbytes = lib.fs4d_render_workspace_bytes(ctypes.byref(info))
    assert 20e6 < nbytes < 400e6


def test_host_errors_without_device(lib):
    """Argument validation happens on the host and maps to featsplat errors."""
    from paper_2503_06161_b200 import _native as N
    from paper_2503_06161_b200.errors import ConfigurationError, DataError
    cloud = N.Cloud()
    cloud.K, cloud.D, cloud.sh_degree = 0, 0, 0
    cam = N.Camera()
    cam.height, cam.width = 16, 16
    cam.K[0], cam.K[4], cam.K[8], cam.K[1] = 10.0, 10.0, 1.0, 0.5   # skewed
    cfg = N.RasterCfg()
    cfg.tile = 16
    info = N.RecordInfo()
    rc = lib.fs4d_render_fwd(ctypes.byref(cloud), ctypes.byref(cam), ctypes.byref(cfg), ctypes.byref(info),
                             None, 0, None, None, None)
    with pytest.raises(DataError):
        N.check(rc)
    cam.K[1] = 0.0
    cfg.tile = 8
    rc = lib.fs4d_render_fwd(ctypes.byref(cloud), ctypes.byref(cam), ctypes.byref(cfg), ctypes.byref(info),
                             None, 0, None, None, None)
    with pytest.raises(ConfigurationError):
        N.check(rc)
