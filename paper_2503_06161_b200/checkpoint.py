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

import struct

import numpy as np

from .errors import FormatError

CHECKPOINT_MAGIC = b"FS4C"
CHECKPOINT_VERSION = 1
# entry kinds (training.py:569-596): array, raw bytes, int64, float64
KIND_ARRAY, KIND_BYTES, KIND_INT, KIND_FLOAT = 0, 1, 2, 3

_U16, _U32, _U64, _I64, _F64 = (struct.Struct(f) for f in ("<H", "<I", "<Q", "<q", "<d"))


def _kind_of(value):
    """Entry kind for a Python / NumPy value (bool and NumPy integers are
    ints; Python and NumPy float64 scalars are floats; anything else is an
    array, including 0-d and non-float64 scalars)."""
    if isinstance(value, (bool, int, np.integer)):
        return KIND_INT
    if isinstance(value, float):
        return KIND_FLOAT
    if isinstance(value, (bytes, bytearray)):
        return KIND_BYTES
    return KIND_ARRAY


def _payload(kind, value):
    if kind == KIND_INT:
        return _I64.pack(int(value))
    if kind == KIND_FLOAT:
        return _F64.pack(float(value))
    if kind == KIND_BYTES:
        return _U64.pack(len(value)) + bytes(value)
    arr = np.ascontiguousarray(value)
    tag = arr.dtype.str.encode("ascii")
    dims = np.asarray(arr.shape, dtype="<u8").tobytes()
    return bytes((len(tag),)) + tag + bytes((arr.ndim,)) + dims + arr.tobytes()


def encode_entries(entries):
    """FS4C bytes: magic, u32 version, u64 count, then the entries in sorted
    name order as (u16 name length, UTF-8 name, i8 kind, payload)."""
    chunks = [CHECKPOINT_MAGIC, _U32.pack(CHECKPOINT_VERSION), _U64.pack(len(entries))]
    for name in sorted(entries):
        key = name.encode("utf-8")
        kind = _kind_of(entries[name])
        chunks += [_U16.pack(len(key)), key, struct.pack("<b", kind), _payload(kind, entries[name])]
    return b"".join(chunks)


def write_entries(path, entries):
    blob = encode_entries(entries)
    with open(path, "wb") as fh:
        fh.write(blob)


class _Cursor:
    """Bounds-checked little-endian reads over an in-memory FS4C image."""

    def __init__(self, blob):
        self.blob = memoryview(blob)
        self.pos = 0

    def take(self, n, what):
        end = self.pos + n
        if end > len(self.blob):
            raise FormatError(f"truncated FS4C data: {what} needs {n} bytes, {len(self.blob) - self.pos} left",
                              offset=self.pos)
        view = self.blob[self.pos:end]
        self.pos = end
        return view

    def unpack(self, st, what):
        return st.unpack(self.take(st.size, what))[0]


def _read_array(cur, name):
    tag = bytes(cur.take(cur.take(1, name)[0], name)).decode("ascii")
    ndim = cur.take(1, name)[0]
    shape = tuple(int(d) for d in np.frombuffer(cur.take(8 * ndim, name), dtype="<u8"))
    dtype = np.dtype(tag)
    count = int(np.prod(shape, dtype=np.int64))
    return np.frombuffer(cur.take(dtype.itemsize * count, name), dtype=dtype).reshape(shape).copy()


_READERS = {
    KIND_INT: lambda cur, name: cur.unpack(_I64, name),
    KIND_FLOAT: lambda cur, name: cur.unpack(_F64, name),
    KIND_BYTES: lambda cur, name: bytes(cur.take(cur.unpack(_U64, name), name)),
    KIND_ARRAY: _read_array,
}


def decode_entries(blob, source="<bytes>"):
    """Inverse of encode_entries; FormatError (byte offset attached) on a bad
    magic, an unsupported version, an unknown kind or truncation
    (training.py:640-674)."""
    cur = _Cursor(blob)
    if bytes(cur.blob[:4]) != CHECKPOINT_MAGIC:
        raise FormatError(f"{source} is not an FS4C checkpoint", offset=0)
    cur.pos = 4
    version = cur.unpack(_U32, "header")
    if version != CHECKPOINT_VERSION:
        raise FormatError(f"FS4C version {version} is not supported (want {CHECKPOINT_VERSION})", offset=4)
    count = cur.unpack(_U64, "header")
    out = {}
    for _ in range(count):
        name = bytes(cur.take(cur.unpack(_U16, "entry name length"), "entry name")).decode("utf-8")
        kind = struct.unpack("<b", cur.take(1, name))[0]
        reader = _READERS.get(kind)
        if reader is None:
            raise FormatError(f"entry {name!r} has unknown kind {kind}", offset=cur.pos)
        out[name] = reader(cur, name)
    return out


def load_entries(path):
    """Entries dict of an FS4C file."""
    with open(path, "rb") as fh:
        return decode_entries(fh.read(), repr(path))


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
