"""Multi-GPU plumbing for the render path.

* Rendering a frame sequence (configs[2]) shards timesteps into contiguous
  blocks, one block per rank; every rank holds a model replica and renders
  its own frames — no data-path collective.
* A data-parallel training step (configs[4]) keeps every gradient of the
  model in ONE flat fp32 buffer (per-Gaussian grads in the a16 order of
  SURVEY §8(e): positions 3, rotations 4, log-scales 3, opacity 1, SH 48
  (colours + higher bands), features 16; then HexPlane planes; then MLP
  weights) so the exchange is a single all-reduce (NCCL over NVLink on the
  GPU box; gloo in the CPU tests).  The 1/world averaging is folded into the
  loss weights, so the collective is a plain SUM.

Process model: one process per GPU (torchrun), torch.distributed for the
plumbing.  Nothing here launches compute.
"""

import numpy as np
import torch

PER_GAUSSIAN = (("positions", 3), ("rotations", 4), ("log_scales", 3), ("opacity_logits", 1),
                ("colors_raw", 3), ("sh_rest", None), ("features", None))


def shard_range(n_items, world, rank):
    """Contiguous block [start, stop) of rank `rank` (np.array_split sizes:
    the first n % world ranks get one extra item)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(int(n_items), int(world))
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def sequence_timesteps(n_frames):
    """configs[2] timesteps t_k = k / (n_frames - 1)."""
    return np.arange(n_frames, dtype=np.float64) / max(n_frames - 1, 1)


def shard_timesteps(n_frames, world, rank):
    lo, hi = shard_range(n_frames, world, rank)
    return sequence_timesteps(n_frames)[lo:hi]


class FlatGrads:
    """One contiguous fp32 buffer with named, shaped views.  Every view starts
    on a 64-byte boundary (`align` floats) so the kernels' vector loads see
    aligned arrays when parameters live in the buffer; the zero padding
    between views rides along in the all-reduce."""

    def __init__(self, specs, device="cuda", align=16):
        self.specs = [(name, tuple(int(s) for s in shape)) for name, shape in specs]
        self.sizes = [int(np.prod(shape)) if len(shape) else 1 for _, shape in self.specs]
        self.offsets = []
        off = 0
        for n in self.sizes:
            self.offsets.append(off)
            off += -(-n // align) * align
        self.numel = int(off)
        self.buffer = torch.zeros(self.numel, dtype=torch.float32, device=device)
        self.views = {}
        for (name, shape), o, n in zip(self.specs, self.offsets, self.sizes):
            self.views[name] = self.buffer[o:o + n].view(shape)

    def __getitem__(self, name):
        return self.views[name]

    def zero_(self):
        self.buffer.zero_()
        return self

    def span(self, first, last):
        """[lo, hi) of the consecutive views first..last; hi is the next
        view's (aligned) offset, or the end of the buffer."""
        names = [n for n, _ in self.specs]
        i, j = names.index(first), names.index(last)
        if j < i:
            raise ValueError("span: views out of order")
        return self.offsets[i], (self.offsets[j + 1] if j + 1 < len(names) else self.numel)

    def allreduce_sum_range(self, lo, hi, group=None, async_op=False):
        """SUM over the group of buffer[lo:hi] (one gradient bucket).  Returns
        the async work handle (async_op=True) or None; no-op when not
        distributed or the range is empty."""
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1 and hi > lo:
            return dist.all_reduce(self.buffer[lo:hi], op=dist.ReduceOp.SUM, group=group, async_op=async_op)
        return None

    def allreduce_sum(self, group=None):
        """In-place SUM over the process group (no-op when not distributed)."""
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
            dist.all_reduce(self.buffer, op=dist.ReduceOp.SUM, group=group)
        return self


def gradient_specs(k, d, sh_degree, plane_shapes, layer_shapes):
    """Flat-buffer layout: per-Gaussian grads, planes, MLP."""
    n_sh = (sh_degree + 1) ** 2 - 1
    specs = []
    for name, width in PER_GAUSSIAN:
        if name == "sh_rest":
            if n_sh:
                specs.append((name, (k, n_sh, 3)))
            continue
        if name == "features":
            specs.append((name, (k, d)))
            continue
        specs.append((name, (k, width) if width > 1 else (k,)))
    for l, level in enumerate(plane_shapes):
        for p, shape in enumerate(level):
            specs.append((f"grid.l{l}.p{p}", tuple(shape)))
    for name, shape in layer_shapes:
        specs.append((name, tuple(shape)))
    return specs
