"""ctypes binding of libfs4d.so (include/fs4d.h) and the error-code map.

The shared library is built in-tree by ``__graft_entry__.build()`` (nvcc,
``-gencode arch=compute_100a,code=sm_100a``).  There is no CPU fallback: if
the library is missing, importing the device path raises immediately.
"""

import ctypes
import os

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfs4d.so")

ABI_VERSION = 1

OK, ERR_CONFIG, ERR_DATA, ERR_NUMERIC, ERR_CONTRACT, ERR_CAPACITY, ERR_DEGENERATE, ERR_CUDA = range(8)

STATUS_WORDS = 32
ST_CODE, ST_BAD_FIELDS, ST_N_VISIBLE, ST_PAIRS_LO, ST_PAIRS_HI = 0, 1, 2, 3, 4
ST_BAD_INDEX, ST_DEGEN_INDEX = 8, 16
ST_ADAM_BAD_SEG, ST_ADAM_BAD_COUNT = 17, 18
ADAM_GATED = -1  # FS4D_ADAM_GATED: the Adam step was skipped because a gated-in call failed
MAX_ADAM_SEGMENTS = 128

FIELD_NAMES = ("positions", "rotations", "log_scales", "opacity_logits",
               "colors_raw", "features", "sh_rest")

MAX_LEVELS = 8
MAX_TRUNK = 16
N_BRANCHES = 4

c_float_p = ctypes.POINTER(ctypes.c_float)
c_int32_p = ctypes.POINTER(ctypes.c_int32)


class Cloud(ctypes.Structure):
    _fields_ = [("K", ctypes.c_int64), ("D", ctypes.c_int32), ("sh_degree", ctypes.c_int32),
                ("positions", ctypes.c_void_p), ("rotations", ctypes.c_void_p),
                ("log_scales", ctypes.c_void_p), ("opacity_logits", ctypes.c_void_p),
                ("colors_raw", ctypes.c_void_p), ("sh_rest", ctypes.c_void_p),
                ("features", ctypes.c_void_p)]


class Camera(ctypes.Structure):
    _fields_ = [("height", ctypes.c_int32), ("width", ctypes.c_int32),
                ("K", ctypes.c_double * 9), ("T", ctypes.c_double * 16)]


class RasterCfg(ctypes.Structure):
    _fields_ = [("tile", ctypes.c_int32), ("with_features", ctypes.c_int32),
                ("z_near", ctypes.c_double), ("lowpass", ctypes.c_double),
                ("alpha_cap", ctypes.c_double), ("alpha_skip", ctypes.c_double),
                ("stop_transmittance", ctypes.c_double), ("background", ctypes.c_double * 3)]


class RecordInfo(ctypes.Structure):
    _fields_ = [("K", ctypes.c_int64), ("height", ctypes.c_int32), ("width", ctypes.c_int32),
                ("D", ctypes.c_int32), ("sh_degree", ctypes.c_int32), ("tile", ctypes.c_int32),
                ("pad_", ctypes.c_int32), ("pair_capacity", ctypes.c_int64)]


class Images(ctypes.Structure):
    _fields_ = [("color", ctypes.c_void_p), ("depth", ctypes.c_void_p),
                ("feature", ctypes.c_void_p), ("alpha", ctypes.c_void_p),
                ("n_contrib", ctypes.c_void_p)]


class ImageGrads(ctypes.Structure):
    _fields_ = [("d_color", ctypes.c_void_p), ("d_depth", ctypes.c_void_p),
                ("d_feature", ctypes.c_void_p), ("d_alpha", ctypes.c_void_p)]


class Projected(ctypes.Structure):
    _fields_ = [("mean2d", ctypes.c_void_p), ("cov2d", ctypes.c_void_p),
                ("conic", ctypes.c_void_p), ("view_depth", ctypes.c_void_p),
                ("radius", ctypes.c_void_p), ("color", ctypes.c_void_p),
                ("opacity", ctypes.c_void_p), ("source_index", ctypes.c_void_p),
                ("tiles_touched", ctypes.c_void_p)]


class HexPlane(ctypes.Structure):
    _fields_ = [("levels", ctypes.c_int32), ("channels", ctypes.c_int32),
                ("res", ((ctypes.c_int32 * 2) * 6) * MAX_LEVELS),
                ("planes", (ctypes.c_void_p * 6) * MAX_LEVELS),
                ("aabb", ctypes.c_double * 6), ("order", ctypes.c_void_p)]


class Linear(ctypes.Structure):
    _fields_ = [("weight", ctypes.c_void_p), ("bias", ctypes.c_void_p),
                ("in_dim", ctypes.c_int32), ("out_dim", ctypes.c_int32), ("relu", ctypes.c_int32)]


class DeformNet(ctypes.Structure):
    _fields_ = [("latent_dim", ctypes.c_int32), ("width", ctypes.c_int32),
                ("depth", ctypes.c_int32), ("feature_dim", ctypes.c_int32),
                ("enable_grid", ctypes.c_int32), ("enable_feature_update", ctypes.c_int32),
                ("trunk", Linear * MAX_TRUNK), ("ext", (Linear * 2) * N_BRANCHES),
                ("head", Linear * N_BRANCHES), ("feat", Linear * 2)]


class AdamSegment(ctypes.Structure):
    _fields_ = [("offset", ctypes.c_int64), ("count", ctypes.c_int64), ("lr", ctypes.c_double),
                ("eps", ctypes.c_double), ("beta1", ctypes.c_double), ("beta2", ctypes.c_double)]


_V, _I32, _I64, _D, _SZ = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_size_t

class DensityConfig(ctypes.Structure):
    _fields_ = [("grad_threshold", ctypes.c_double), ("percent_dense", ctypes.c_double),
                ("prune_opacity", ctypes.c_double), ("split_factor", ctypes.c_double),
                ("extent", ctypes.c_double)]


# symbol -> (restype, argtypes); every entry point declared in include/fs4d.h
SIGNATURES = {
    "fs4d_abi_version": (ctypes.c_int, []),
    "fs4d_last_error": (ctypes.c_char_p, []),
    "fs4d_build_info": (ctypes.c_char_p, []),
    "fs4d_status_reset": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    "fs4d_status_merge": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p]),
    "fs4d_profile_enable": (ctypes.c_int, [ctypes.c_int]),
    "fs4d_profile_collect": (ctypes.c_int, [ctypes.POINTER(ctypes.c_double),
                                            ctypes.POINTER(ctypes.c_int64), ctypes.c_int32]),
    "fs4d_deform_workspace_bytes": (ctypes.c_size_t, [ctypes.POINTER(DeformNet), ctypes.c_int64]),
    "fs4d_deform_cache_bytes": (ctypes.c_size_t, [ctypes.POINTER(DeformNet), ctypes.POINTER(HexPlane),
                                                  ctypes.c_int64]),
    "fs4d_deform_fwd": (ctypes.c_int, [ctypes.POINTER(Cloud), ctypes.POINTER(HexPlane),
                                       ctypes.POINTER(DeformNet), ctypes.c_double,
                                       ctypes.POINTER(Cloud), ctypes.c_void_p, ctypes.c_size_t,
                                       ctypes.c_void_p, ctypes.c_size_t,
                                       ctypes.c_void_p, ctypes.c_void_p]),
    "fs4d_deform_bwd": (ctypes.c_int, [ctypes.POINTER(Cloud), ctypes.POINTER(HexPlane),
                                       ctypes.POINTER(DeformNet), ctypes.c_double,
                                       ctypes.c_void_p, ctypes.c_size_t,
                                       ctypes.POINTER(Cloud), ctypes.POINTER(Cloud),
                                       ctypes.POINTER(DeformNet), ctypes.POINTER(HexPlane),
                                       ctypes.c_int32, ctypes.c_void_p, ctypes.c_size_t,
                                       ctypes.c_void_p, ctypes.c_void_p]),
    "fs4d_sum_buffers": (ctypes.c_int, [_V, ctypes.POINTER(ctypes.c_void_p), _I32, _I64, _I32, _V]),
    "fs4d_hexplane_query": (ctypes.c_int, [ctypes.POINTER(HexPlane), _V, _I64, _D, _V, _V]),
    "fs4d_hexplane_query_backward": (ctypes.c_int, [ctypes.POINTER(HexPlane), _V, _I64, _D, _V,
                                                    ctypes.POINTER(HexPlane), _V, _I32, _V]),
    "fs4d_linear_forward": (ctypes.c_int, [_V, _I64, ctypes.POINTER(Linear), _V, _V, _V]),
    "fs4d_linear_backward_workspace_bytes": (_SZ, [_I64, _I32, _I32]),
    "fs4d_linear_backward": (ctypes.c_int, [_V, _V, _I64, ctypes.POINTER(Linear), _V, _V, _V, _V, _I32, _V, _SZ,
                                            _V]),
    "fs4d_render_tile_alphas": (ctypes.c_int, [ctypes.POINTER(RecordInfo), _V, _SZ, ctypes.POINTER(RasterCfg), _V,
                                               _I64, _I32, _I32, _I32, _I32, _V, _V, _V, _V]),
    "fs4d_composite_weights": (ctypes.c_int, [_V, _I64, _I64, _D, _V, _V, _V, _V, _V]),
    "fs4d_deform_bwd_deterministic": (ctypes.c_int, [ctypes.POINTER(Cloud), ctypes.POINTER(HexPlane),
                                                     ctypes.POINTER(DeformNet), ctypes.c_double,
                                                     ctypes.c_void_p, ctypes.c_size_t,
                                                     ctypes.POINTER(Cloud), ctypes.POINTER(Cloud),
                                                     ctypes.POINTER(DeformNet), ctypes.POINTER(HexPlane),
                                                     ctypes.c_int32, ctypes.c_void_p, ctypes.c_size_t,
                                                     ctypes.c_void_p, ctypes.c_size_t,
                                                     ctypes.c_void_p, ctypes.c_void_p]),
    "fs4d_deform_bwd_split": (ctypes.c_int, [ctypes.POINTER(Cloud), ctypes.POINTER(HexPlane),
                                             ctypes.POINTER(DeformNet), ctypes.c_double,
                                             ctypes.c_void_p, ctypes.c_size_t,
                                             ctypes.POINTER(Cloud), ctypes.POINTER(Cloud),
                                             ctypes.POINTER(DeformNet), ctypes.POINTER(HexPlane),
                                             ctypes.c_int32, ctypes.c_void_p, ctypes.c_size_t,
                                             ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p,
                                             ctypes.c_void_p, ctypes.c_void_p]),
    "fs4d_deform_bwd_det_workspace_bytes": (ctypes.c_size_t, [ctypes.POINTER(DeformNet), ctypes.POINTER(HexPlane)]),
    "fs4d_l1_loss_grad": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                         ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32,
                                         ctypes.c_int32, ctypes.c_double, ctypes.c_double,
                                         ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                         ctypes.c_void_p]),
    "fs4d_photometric_workspace_bytes": (_SZ, [_I32, _I32]),
    "fs4d_photometric_loss_grad": (ctypes.c_int, [_V, _V, _V, _V, _V, _V, _I32, _I32, _D, _D, _V, _V, _V,
                                                  _V, _V, _SZ, _V]),
    "fs4d_l1": (ctypes.c_int, [_V, _V, _I64, _D, _V, _V, _V]),
    "fs4d_adam_step": (ctypes.c_int, [_V, _V, _V, _V, _V, ctypes.POINTER(AdamSegment), _I32, _V, _V]),
    "fs4d_adam_step_masked": (ctypes.c_int, [_V, _V, _V, _V, _V, ctypes.POINTER(AdamSegment),
                                             ctypes.POINTER(ctypes.c_int32), _I32, _V, _V]),
    "fs4d_tv_loss_grad": (ctypes.c_int, [ctypes.POINTER(HexPlane), ctypes.POINTER(HexPlane), _D, _I32, _V, _V]),
    "fs4d_resize_bilinear": (ctypes.c_int, [_V, _I32, _I32, _I32, _V, _I32, _I32, _V]),
    "fs4d_resize_workspace_bytes": (_SZ, [_I32, _I32, _I32]),
    "fs4d_resize_bilinear_backward": (ctypes.c_int, [_V, _I32, _I32, _I32, _V, _I32, _I32, _V, _SZ, _V]),
    "fs4d_decoder_workspace_bytes": (_SZ, [_I32, _I32, _I32, _I32, _I32, _I32]),
    "fs4d_decode_features": (ctypes.c_int, [_V, _I32, _I32, _I32, _V, _V, _I32, _I32, _I32, _V, _V, _V]),
    "fs4d_decode_features_backward": (ctypes.c_int, [_V, _V, _V, _I32, _I32, _I32, _I32, _I32, _I32, _V, _V, _V,
                                                     _I32, _V, _SZ, _V]),
    "fs4d_decoder_feature_loss": (ctypes.c_int, [_V, _I32, _I32, _I32, _V, _V, _I32, _V, _I32, _I32, _D, _V, _V,
                                                 _V, _I32, _V, _V, _SZ, _V]),
    "fs4d_grad_stats_add": (ctypes.c_int, [_V, _V, _V, _V, _I64, _V, _V]),
    "fs4d_density_workspace_bytes": (_SZ, [_I64, _I64]),
    "fs4d_density_classify": (ctypes.c_int, [ctypes.POINTER(Cloud), _V, _V, ctypes.POINTER(DensityConfig), _I32,
                                             _I64, _V, _V, _SZ, _V, _V]),
    "fs4d_density_apply": (ctypes.c_int, [ctypes.POINTER(Cloud), _V, ctypes.POINTER(DensityConfig), _I64, _I32,
                                          _I32, _I32, ctypes.POINTER(Cloud), _V, _V, _V, _V, _I32, _I32,
                                          ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_void_p),
                                          ctypes.POINTER(ctypes.c_int32), _V, _SZ, _V, _V]),
    "fs4d_reset_opacity": (ctypes.c_int, [_V, _I64, _D, _V]),
    "fs4d_locality_order_workspace_bytes": (_SZ, [_I64]),
    "fs4d_locality_order": (ctypes.c_int, [_V, _I64, ctypes.POINTER(ctypes.c_double), _V, _V, _SZ, _V]),
    "fs4d_render_workspace_bytes": (ctypes.c_size_t, [ctypes.POINTER(RecordInfo)]),
    "fs4d_render_fwd": (ctypes.c_int, [ctypes.POINTER(Cloud), ctypes.POINTER(Camera),
                                       ctypes.POINTER(RasterCfg), ctypes.POINTER(RecordInfo),
                                       ctypes.c_void_p, ctypes.c_size_t, ctypes.POINTER(Images),
                                       ctypes.c_void_p, ctypes.c_void_p]),
    "fs4d_render_bwd": (ctypes.c_int, [ctypes.POINTER(Cloud), ctypes.POINTER(Camera),
                                       ctypes.POINTER(RasterCfg), ctypes.POINTER(RecordInfo),
                                       ctypes.c_void_p, ctypes.c_size_t, ctypes.POINTER(ImageGrads),
                                       ctypes.POINTER(Cloud), ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_void_p]),
    "fs4d_render_bwd_deterministic": (ctypes.c_int, [ctypes.POINTER(Cloud), ctypes.POINTER(Camera),
                                                     ctypes.POINTER(RasterCfg), ctypes.POINTER(RecordInfo),
                                                     ctypes.c_void_p, ctypes.c_size_t, ctypes.POINTER(ImageGrads),
                                                     ctypes.POINTER(Cloud), ctypes.c_void_p, ctypes.c_void_p,
                                                     ctypes.c_void_p, ctypes.c_size_t,
                                                     ctypes.c_void_p, ctypes.c_void_p]),
    "fs4d_render_bwd_det_workspace_bytes": (ctypes.c_size_t, [ctypes.POINTER(RecordInfo)]),
    "fs4d_render_export_projected": (ctypes.c_int, [ctypes.POINTER(RecordInfo), ctypes.c_void_p,
                                                    ctypes.c_size_t, ctypes.POINTER(Projected),
                                                    ctypes.c_void_p]),
    "fs4d_render_export_tiles": (ctypes.c_int, [ctypes.POINTER(RecordInfo), ctypes.c_void_p,
                                                ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p,
                                                ctypes.c_int64, ctypes.c_void_p]),
}

_lib = None


def load():
    """Load libfs4d.so once; raise loudly if it is missing or mismatched."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (restype, argtypes) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = restype
        fn.argtypes = argtypes
    if lib.fs4d_abi_version() != ABI_VERSION:
        raise ImportError("libfs4d ABI version mismatch")
    _lib = lib
    return lib


_EXC = {
    ERR_CONFIG: errors.ConfigurationError,
    ERR_DATA: errors.DataError,
    ERR_NUMERIC: errors.NumericalError,
    ERR_CONTRACT: errors.ContractViolation,
    ERR_DEGENERATE: errors.DegenerateRotationError,
}


class CapacityError(errors.FeatsplatError):
    """Pair buffer overflow; the caller grows the record and retries."""


def check(rc):
    """Raise the featsplat exception matching a host-side return code."""
    if rc == OK:
        return
    msg = load().fs4d_last_error().decode(errors="replace")
    if rc == ERR_CAPACITY:
        raise CapacityError(msg)
    raise _EXC.get(rc, RuntimeError)(msg)


def raise_device_status(st):
    """Turn a read-back status block (sequence of ints) into an exception."""
    code = int(st[ST_CODE])
    if code == OK:
        return
    if code == ERR_NUMERIC:
        mask = int(st[ST_BAD_FIELDS])
        for f, name in enumerate(FIELD_NAMES):
            if mask & (1 << f):
                raise errors.NumericalError(
                    f"non-finite {name} for Gaussian indices [{int(st[ST_BAD_INDEX + f])}]")
        raise errors.NumericalError("non-finite snapshot parameters")
    if code == ERR_DEGENERATE:
        raise errors.DegenerateRotationError(
            f"quaternion norm below 1e-12 (index {int(st[ST_DEGEN_INDEX])})")
    if code == ERR_CAPACITY:
        pairs = (int(st[ST_PAIRS_HI]) << 32) | (int(st[ST_PAIRS_LO]) & 0xFFFFFFFF)
        raise CapacityError(f"tile pair buffer too small: {pairs} pairs")
    raise RuntimeError(f"libfs4d device status {code}")
