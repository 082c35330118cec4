"""B200-native FE-4DGS per-frame render path (arXiv 2503.06161).

Drop-in for the reference package's render path (featsplat: deformation,
hexplane query, rasterizer and their backward passes).  Host code is NumPy /
PyTorch; all math runs in libfs4d.so, hand-written CUDA for sm_100a behind a
C ABI (include/fs4d.h).  There is no CPU fallback.
"""

__version__ = "0.1.0"

from .errors import (ConfigurationError, ContractViolation, DataError, DegenerateRotationError,
                     FeatsplatError, FormatError, NumericalError)
from .gaussians import CameraFrame, GaussianCloud, logit, scene_aabb, sigmoid
from .hexplane import (PLANE_AXES, HexPlaneConfig, HexPlaneField, query, query_backward, query_with_cache,
                       tv_backward, tv_loss)
from .numerics import LinearLayer, linear_layer, mlp_backward, mlp_forward
from .deformation import (BRANCH_DIMS, BRANCHES, DeformationConfig, DeformationNet, decode_branches,
                          decode_hidden, deform, deform_backward, deform_with_cache, update_semantics)
from .rasterizer import (ProjectedGaussians, RasterConfig, RasterRecord, RenderOutput, SnapshotGrads, TileRecord,
                         bin_tiles, project, render, render_backward)

__all__ = [
    "CameraFrame", "GaussianCloud", "HexPlaneConfig", "HexPlaneField", "PLANE_AXES",
    "DeformationConfig", "DeformationNet", "deform", "deform_with_cache", "deform_backward",
    "RasterConfig", "ProjectedGaussians", "RenderOutput", "SnapshotGrads", "project", "bin_tiles",
    "render", "render_backward", "LinearLayer", "linear_layer", "sigmoid", "logit", "scene_aabb",
    "query", "query_with_cache", "query_backward", "tv_loss", "tv_backward", "mlp_forward", "mlp_backward",
    "decode_hidden", "decode_branches", "update_semantics", "RasterRecord", "TileRecord",
    "BRANCHES", "BRANCH_DIMS", "FeatsplatError", "ConfigurationError", "DataError", "FormatError",
    "ContractViolation", "NumericalError", "DegenerateRotationError", "__version__",
]
