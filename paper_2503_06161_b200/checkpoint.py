"""FS4C checkpoint container (training.py:44-45, 569-706) read and written
from device buffers -- SURVEY §8(f) row 4.

The container codec is the reference's byte format: magic "FS4C", u32
version 1, u64 entry count, then name-sorted entries (u16 name length, name,
i8 kind, payload: i64 int | f64 float | u64 length + bytes | dtype string,
ndim, u64 dims, C-order data).  A file written here is byte-identical to the
reference's for the same entries (tests/test_checkpoint_cpu.py pins it
against a file the reference wrote).

``train_state_entries`` / ``load_train_state`` map a device TrainStep (flat
fp32 parameter / Adam buffers, train.py) to the reference's entry names
(cloud.<field>, grid.l<l>.p<p>, net.<stack>.<i>.weight|bias, decoder.*,
adam.<name>.m|v|step, stats.*), upcasting fp32 to the reference's float64
(exact) on save and rounding to fp32 on load.  Everything that is not model
state (meta.config INI, meta.rng, frame schedule) belongs to the training
driver, which is out of scope; callers pass those entries through `meta`.
"""

import io
import struct

import numpy as np

from .errors import FormatError

CHECKPOINT_MAGIC = b"FS4C"
CHECKPOINT_VERSION = 1
_KIND_ARRAY, _KIND_BYTES, _KIND_INT, _KIND_FLOAT = 0, 1, 2, 3


def _write_entry(buf, name, value):
    nb = name.encode()
    buf.write(struct.pack("<H", len(nb)))
    buf.write(nb)
    if isinstance(value, (bool, int, np.integer)):
        buf.write(struct.pack("<bq", _KIND_INT, int(value)))
    elif isinstance(value, float):
        buf.write(struct.pack("<bd", _KIND_FLOAT, value))
    elif isinstance(value, bytes):
        buf.write(struct.pack("<bQ", _KIND_BYTES, len(value)))
        buf.write(value)
    else:
        arr = np.ascontiguousarray(value)
        dt = arr.dtype.str.encode()
        buf.write(struct.pack("<bB", _KIND_ARRAY, len(dt)))
        buf.write(dt)
        buf.write(struct.pack("<B", arr.ndim))
        for dim in arr.shape:
            buf.write(struct.pack("<Q", dim))
        buf.write(arr.tobytes(order="C"))


def encode_entries(entries):
    buf = io.BytesIO()
    buf.write(CHECKPOINT_MAGIC)
    buf.write(struct.pack("<IQ", CHECKPOINT_VERSION, len(entries)))
    for name in sorted(entries):
        _write_entry(buf, name, entries[name])
    return buf.getvalue()


def write_entries(path, entries):
    with open(path, "wb") as fh:
        fh.write(encode_entries(entries))


def _read_exact(fh, n, what):
    data = fh.read(n)
    if len(data) != n:
        raise FormatError(f"truncated checkpoint while reading {what}", offset=fh.tell())
    return data


def load_entries(path):
    """Entries dict of an FS4C file; FormatError (with byte offset) on a
    bad magic, version, kind or a truncated file (training.py:640-674)."""
    with open(path, "rb") as fh:
        if fh.read(4) != CHECKPOINT_MAGIC:
            raise FormatError(f"bad checkpoint magic in {path!r}", offset=0)
        version, count = struct.unpack("<IQ", _read_exact(fh, 12, "header"))
        if version != CHECKPOINT_VERSION:
            raise FormatError(f"unsupported checkpoint version {version}", offset=4)
        entries = {}
        for _ in range(count):
            (nlen,) = struct.unpack("<H", _read_exact(fh, 2, "name length"))
            name = _read_exact(fh, nlen, "name").decode()
            (kind,) = struct.unpack("<b", _read_exact(fh, 1, "kind"))
            if kind == _KIND_INT:
                (entries[name],) = struct.unpack("<q", _read_exact(fh, 8, name))
            elif kind == _KIND_FLOAT:
                (entries[name],) = struct.unpack("<d", _read_exact(fh, 8, name))
            elif kind == _KIND_BYTES:
                (blen,) = struct.unpack("<Q", _read_exact(fh, 8, name))
                entries[name] = _read_exact(fh, blen, name)
            elif kind == _KIND_ARRAY:
                (dlen,) = struct.unpack("<B", _read_exact(fh, 1, name))
                dtype = np.dtype(_read_exact(fh, dlen, name).decode())
                (ndim,) = struct.unpack("<B", _read_exact(fh, 1, name))
                shape = struct.unpack(f"<{ndim}Q", _read_exact(fh, 8 * ndim, name))
                n = int(np.prod(shape, dtype=np.int64)) if ndim else 1
                raw = _read_exact(fh, dtype.itemsize * n, name)
                entries[name] = np.frombuffer(raw, dtype=dtype).reshape(shape).copy()
            else:
                raise FormatError(f"unknown entry kind {kind} for {name!r}", offset=fh.tell())
        return entries


# ---------------------------------------------------------------------------
# device training state <-> entries
# ---------------------------------------------------------------------------
def _host64(t):
    return t.detach().cpu().numpy().astype(np.float64)


def _param_name(name):
    """Flat-buffer spec name -> checkpoint entry name (training.py:573-596)."""
    if name.startswith(("grid.", "net.", "decoder.")):
        return name
    return f"cloud.{name}"


def train_state_entries(step, meta=None, stats=None):
    """Entries of a device TrainStep with an attached optimizer: every
    parameter array, its Adam moments and step count, optional grad stats
    (density.ViewspaceGradStats) and caller-supplied meta entries."""
    if step.optimizer is None:
        raise ValueError("attach_optimizer() first: the checkpoint holds Adam state")
    entries = dict(meta or {})
    steps = step.optimizer.steps.cpu().numpy()
    params = step.params
    for i, (name, shape) in enumerate(step.specs):
        off, n = params.offsets[i], params.sizes[i]
        entries[_param_name(name)] = _host64(params.buffer[off:off + n]).reshape(shape)
        entries[f"adam.{name}.m"] = _host64(step.optimizer.m[off:off + n]).reshape(shape)
        entries[f"adam.{name}.v"] = _host64(step.optimizer.v[off:off + n]).reshape(shape)
        entries[f"adam.{name}.step"] = int(steps[i])
    if stats is not None:
        entries["stats.accum"] = _host64(stats.accum) if hasattr(stats.accum, "cpu") else np.asarray(stats.accum)
        entries["stats.count"] = _host64(stats.count) if hasattr(stats.count, "cpu") else np.asarray(stats.count)
    entries.setdefault("meta.iteration", int(step.iteration))
    return entries


def save_train_state(step, path, meta=None, stats=None):
    write_entries(path, train_state_entries(step, meta, stats))


def load_train_state(step, path_or_entries):
    """Fill a TrainStep (optimizer attached, same shapes) from an FS4C file
    or entries dict; returns the entries (meta.* for the caller)."""
    import torch

    entries = load_entries(path_or_entries) if isinstance(path_or_entries, str) else path_or_entries
    if step.optimizer is None:
        raise ValueError("attach_optimizer() first")
    params = step.params
    steps = []
    for i, (name, shape) in enumerate(step.specs):
        off, n = params.offsets[i], params.sizes[i]
        src = np.asarray(entries[_param_name(name)], dtype=np.float64)
        if tuple(src.shape) != tuple(shape):
            raise FormatError(f"checkpoint entry {name} has shape {src.shape}, expected {shape}")
        dev = params.buffer.device
        params.buffer[off:off + n].copy_(torch.as_tensor(src.reshape(-1), dtype=torch.float32, device=dev))
        for tag, buf in (("m", step.optimizer.m), ("v", step.optimizer.v)):
            key = f"adam.{name}.{tag}"
            arr = np.asarray(entries[key], dtype=np.float64).reshape(-1) if key in entries else np.zeros(n)
            buf[off:off + n].copy_(torch.as_tensor(arr, dtype=torch.float32, device=dev))
        steps.append(int(entries.get(f"adam.{name}.step", 0)))
    step.optimizer.steps.copy_(torch.tensor(steps, dtype=torch.int32))
    if "meta.iteration" in entries:
        step.iteration = int(entries["meta.iteration"])
    return entries
