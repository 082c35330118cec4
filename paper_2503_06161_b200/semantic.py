"""semantic.py API of the reference on device: the
corner-aligned bilinear resize and its adjoint (semantic.py:82-123), the
pointwise feature decoder with its backward (semantic.py:126-168), the
feature L1 loss (semantic.py:171-181), and the FE4D teacher-feature
container (semantic.py:17-75).

Every function takes the reference's float64 NumPy arrays (returns NumPy) or
fp32 CUDA tensors (returns CUDA tensors, no host round trip).  The math runs
in libfs4d (csrc/train_ops.cu); there is no CPU fallback.
"""

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .device import _p, _stream, as_device, to_host
from .errors import ConfigurationError, FormatError

MAGIC = b"FE4D"      # semantic.py:17
FORMAT_VERSION = 1   # semantic.py:18


# ---------------------------------------------------------------------------
# FE4D feature container (semantic.py:17-75): host file format
# ---------------------------------------------------------------------------
# The 18-byte header as one packed little-endian record; the payload follows
# as C*H*W little-endian float32 in channel-major order.
_FE4D_HEADER = np.dtype([("magic", "S4"), ("version", "<u2"), ("channels", "<u4"),
                         ("height", "<u4"), ("width", "<u4")])
assert _FE4D_HEADER.itemsize == 18


class FeatureMap:
    """Teacher feature map, float32 [C, H, W] (semantic.py:21-46)."""

    __slots__ = ("data",)

    def __init__(self, data):
        arr = np.asarray(data)
        if arr.ndim != 3 or 0 in arr.shape:
            raise ConfigurationError("feature map must be [C, H, W] with positive dims")
        self.data = np.ascontiguousarray(arr, dtype=np.float32)

    def __repr__(self):
        return f"FeatureMap(channels={self.channels}, height={self.height}, width={self.width})"

    def __eq__(self, other):
        return isinstance(other, FeatureMap) and np.array_equal(self.data, other.data)

    channels = property(lambda self: int(self.data.shape[0]))
    height = property(lambda self: int(self.data.shape[1]))
    width = property(lambda self: int(self.data.shape[2]))

    def hwc(self):
        """Float64 [H, W, C] copy for arithmetic."""
        return self.data.transpose(1, 2, 0).astype(np.float64)

    def to_device(self, device="cuda"):
        """[H, W, C] fp32 CUDA tensor (the layout the decoder loss reads)."""
        return torch.as_tensor(self.data, device=device).permute(1, 2, 0).contiguous()


def save_feature_map(path, fmap):
    """Header record + float32 payload (semantic.py:49-55)."""
    head = np.zeros((), dtype=_FE4D_HEADER)
    head["magic"], head["version"] = MAGIC, FORMAT_VERSION
    head["channels"], head["height"], head["width"] = fmap.data.shape
    with open(path, "wb") as fh:
        fh.write(head.tobytes())
        fh.write(np.asarray(fmap.data, dtype="<f4").tobytes())


def load_feature_map(path):
    """Parse an FE4D file; every malformed case is a FormatError carrying the
    byte offset where the file stops making sense (semantic.py:58-75)."""
    blob = memoryview(open(path, "rb").read())
    size = len(blob)
    if bytes(blob[:4]) != MAGIC:
        raise FormatError(f"{path!r} is not an FE4D feature file", offset=0)
    if size < _FE4D_HEADER.itemsize:
        raise FormatError(f"{path!r}: header cut short after {size} bytes", offset=size)
    head = np.frombuffer(blob, dtype=_FE4D_HEADER, count=1)[0]
    if int(head["version"]) != FORMAT_VERSION:
        raise FormatError(f"FE4D version {int(head['version'])} is not supported (want {FORMAT_VERSION})",
                          offset=4)
    shape = (int(head["channels"]), int(head["height"]), int(head["width"]))
    want = _FE4D_HEADER.itemsize + 4 * shape[0] * shape[1] * shape[2]
    if size != want:
        raise FormatError(f"{path!r}: file is {size} bytes but its header implies {want}", offset=min(size, want))
    return FeatureMap(np.frombuffer(blob, dtype="<f4", offset=_FE4D_HEADER.itemsize).reshape(shape).copy())


# ---------------------------------------------------------------------------
# bilinear resize (semantic.py:82-123)
# ---------------------------------------------------------------------------
def _hwc(x, what):
    t, host = as_device(x)
    if t.dim() != 3:
        raise ConfigurationError(f"{what} must be [H, W, C], got {tuple(t.shape)}")
    return t, host


def resize_bilinear(img, out_hw):
    """Resize [H, W, C] to out_hw with corner-aligned bilinear interpolation."""
    t, host = _hwc(img, "image")
    hi, wi, c = t.shape
    ho, wo = int(out_hw[0]), int(out_hw[1])
    out = torch.empty(ho, wo, c, dtype=torch.float32, device=t.device)
    N.check(N.load().fs4d_resize_bilinear(_p(t), hi, wi, c, _p(out), ho, wo, _stream()))
    return to_host(out, host)


def resize_bilinear_backward(d_out, in_hw):
    """Adjoint of resize_bilinear (a deterministic gather instead of np.add.at)."""
    t, host = _hwc(d_out, "d_out")
    ho, wo, c = t.shape
    hi, wi = int(in_hw[0]), int(in_hw[1])
    lib = N.load()
    ws = torch.empty(max(int(lib.fs4d_resize_workspace_bytes(ho, wi, c)), 1), dtype=torch.uint8, device=t.device)
    out = torch.empty(hi, wi, c, dtype=torch.float32, device=t.device)
    N.check(lib.fs4d_resize_bilinear_backward(_p(t), ho, wo, c, _p(out), hi, wi, _p(ws), ws.numel(), _stream()))
    return to_host(out, host)


# ---------------------------------------------------------------------------
# pointwise decoder (semantic.py:126-168)
# ---------------------------------------------------------------------------
@dataclass
class PointwiseDecoder:
    """Per-pixel affine map from rendered channels N to teacher channels C_t."""

    weight: object  # [C_t, N]
    bias: object    # [C_t]

    @classmethod
    def create(cls, teacher_channels, rendered_channels, rng):
        bound = np.sqrt(6.0 / rendered_channels)
        return cls(weight=rng.uniform(-bound, bound, size=(teacher_channels, rendered_channels)),
                   bias=np.zeros(teacher_channels))

    def param_arrays(self):
        return {"decoder.weight": self.weight, "decoder.bias": self.bias}


def _decoder_args(decoder, rendered):
    r, host = _hwc(rendered, "rendered")
    w, _ = as_device(decoder.weight)
    b, _ = as_device(decoder.bias)
    if w.dim() != 2 or r.shape[2] != w.shape[1]:
        raise ConfigurationError(f"rendered channels {r.shape[2]} != decoder input {w.shape[1] if w.dim() == 2 else '?'}")
    return r, w, b, host


def decode_features(decoder, rendered, out_hw):
    out, _ = decode_features_with_cache(decoder, rendered, out_hw)
    return out


def decode_features_with_cache(decoder, rendered, out_hw):
    """Bilinear resize of the rendered [H, W, N] map, then W v + b per pixel."""
    r, w, b, host = _decoder_args(decoder, rendered)
    hi, wi, n = r.shape
    ct = w.shape[0]
    ho, wo = int(out_hw[0]), int(out_hw[1])
    out = torch.empty(ho, wo, ct, dtype=torch.float32, device=r.device)
    resized = torch.empty(ho, wo, n, dtype=torch.float32, device=r.device)
    N.check(N.load().fs4d_decode_features(_p(r), hi, wi, n, _p(w), _p(b), ct, ho, wo, _p(out), _p(resized),
                                          _stream()))
    return to_host(out, host), {"resized": resized, "in_hw": (hi, wi), "host": host}


def _decoder_workspace(hi, wi, n, ho, wo, ct, device):
    nbytes = int(N.load().fs4d_decoder_workspace_bytes(hi, wi, n, ho, wo, ct))
    return torch.empty(max(nbytes, 1), dtype=torch.uint8, device=device)


def decode_features_backward(decoder, cache, d_out):
    """Returns (d_rendered, d_weight, d_bias) (semantic.py:161-168)."""
    d, _ = _hwc(d_out, "d_out")
    resized = cache["resized"]
    host = cache.get("host", True)
    w, _ = as_device(decoder.weight)
    hi, wi = cache["in_hw"]
    ho, wo, ct = d.shape
    n = resized.shape[2]
    dev = d.device
    d_rendered = torch.empty(hi, wi, n, dtype=torch.float32, device=dev)
    dw = torch.empty(ct, n, dtype=torch.float32, device=dev)
    db = torch.empty(ct, dtype=torch.float32, device=dev)
    ws = _decoder_workspace(hi, wi, n, ho, wo, ct, dev)
    N.check(N.load().fs4d_decode_features_backward(_p(d), _p(resized), _p(w), hi, wi, n, ct, ho, wo, _p(d_rendered),
                                                   _p(dw), _p(db), 0, _p(ws), ws.numel(), _stream()))
    return to_host(d_rendered, host), to_host(dw, host), to_host(db, host)


class DecoderLoss:
    """Fused decode -> feature L1 -> backward (training.py:497-505 with
    semantic.py:145-181) for the training step: the decoded map and its
    gradient never reach HBM.  Device tensors only."""

    def __init__(self, device="cuda"):
        self.device = device
        self.ws = None

    def __call__(self, weight, bias, rendered, teacher, lam, d_rendered, d_weight, d_bias, loss, accumulate=False):
        hi, wi, n = rendered.shape
        ho, wo, ct = teacher.shape
        need = int(N.load().fs4d_decoder_workspace_bytes(hi, wi, n, ho, wo, ct))
        if self.ws is None or self.ws.numel() < need:
            self.ws = torch.empty(max(need, 1), dtype=torch.uint8, device=self.device)
        N.check(N.load().fs4d_decoder_feature_loss(_p(rendered), hi, wi, n, _p(weight), _p(bias), ct, _p(teacher),
                                                   ho, wo, float(lam), _p(d_rendered), _p(d_weight), _p(d_bias),
                                                   int(bool(accumulate)), _p(loss), _p(self.ws), self.ws.numel(),
                                                   _stream()))


# ---------------------------------------------------------------------------
# feature loss (semantic.py:171-181)
# ---------------------------------------------------------------------------
def _pair(pred, gt):
    p, host = as_device(pred)
    g, _ = as_device(gt)
    if tuple(p.shape) != tuple(g.shape):
        raise ConfigurationError(f"shape mismatch: {tuple(p.shape)} vs {tuple(g.shape)}")
    return p, g, host


def feature_loss(pred, gt):
    """Mean over pixels of the channel-summed L1 difference."""
    p, g, _ = _pair(pred, gt)
    h, w = p.shape[0], p.shape[1]
    loss = torch.zeros(1, dtype=torch.float64, device=p.device)
    N.check(N.load().fs4d_l1(_p(p), _p(g), p.numel(), 1.0 / (h * w), None, _p(loss), _stream()))
    return float(loss.item())


def feature_loss_backward(pred, gt):
    p, g, host = _pair(pred, gt)
    h, w = p.shape[0], p.shape[1]
    grad = torch.empty_like(p)
    N.check(N.load().fs4d_l1(_p(p), _p(g), p.numel(), 1.0 / (h * w), _p(grad), None, _stream()))
    return to_host(grad, host)
