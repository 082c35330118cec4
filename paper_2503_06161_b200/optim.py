"""Adam over device parameters (numerics.py:119-199, training.py:46-47,
365-376, 431-442) -- SURVEY §8(f) row 1.

* ``FlatAdam`` is the training path: every parameter array of the model is a
  segment of ONE flat fp32 buffer (the same layout as the all-reduced
  gradient buffer, parallel.FlatGrads), so the whole optimizer step is two
  kernel launches (non-finite check + update) for all ~50 arrays, each
  segment with its own learning rate, eps and Adam step count exactly as the
  reference keeps one AdamState per array.
* ``numerics.adam_step`` (reference signature) runs the same kernel on a
  single array.

The learning-rate schedule itself is host scalar arithmetic
(``numerics.lr_at_step``), evaluated once per step per group.
"""

import ctypes

import numpy as np
import torch

from . import _native as N
from .device import StatusBlock, _p, _stream
from .errors import ConfigurationError, NumericalError

GAUSSIAN_ADAM_EPS = 1e-15  # training.py:46
NETWORK_ADAM_EPS = 1e-8    # training.py:47


def adam_eps(name):
    """training.py:366-367: dotted names (grid./net./decoder.) are network params."""
    return GAUSSIAN_ADAM_EPS if "." not in name else NETWORK_ADAM_EPS


def schedule_key(name):
    """training.py:370-377."""
    for prefix in ("grid", "net", "decoder"):
        if name.startswith(prefix + "."):
            return prefix
    return name


class FlatAdam:
    """Multi-tensor Adam over a flat fp32 parameter buffer.

    specs: [(name, shape)] in buffer order (parallel.gradient_specs layout).
    params: the flat fp32 CUDA parameter buffer (updated in place).
    offsets: start of each array in the buffer (FlatGrads.offsets, which pads
    every array to 64 bytes); contiguous when None.
    """

    def __init__(self, specs, params, beta1=0.9, beta2=0.999, eps_of=adam_eps, offsets=None):
        self.specs = [(n, tuple(int(s) for s in sh)) for n, sh in specs]
        if len(self.specs) > N.MAX_ADAM_SEGMENTS:
            raise ConfigurationError(f"at most {N.MAX_ADAM_SEGMENTS} parameter arrays per Adam call")
        self.params = params
        self.m = torch.zeros_like(params)
        self.v = torch.zeros_like(params)
        self.steps = torch.zeros(len(self.specs), dtype=torch.int32, device=params.device)
        self.status = StatusBlock(params.device)
        self.status.reset()
        self.segs = (N.AdamSegment * max(len(self.specs), 1))()
        off = 0
        for i, (name, shape) in enumerate(self.specs):
            n = int(np.prod(shape)) if shape else 1
            if offsets is not None:
                off = int(offsets[i])
            s = self.segs[i]
            s.offset, s.count = off, n
            s.eps, s.beta1, s.beta2 = float(eps_of(name)), float(beta1), float(beta2)
            s.lr = 1.0
            off += n
            if off > params.numel():
                raise ConfigurationError(f"Adam segment {name} ends at {off}, buffer has {params.numel()}")
        self.names = [n for n, _ in self.specs]

    def step(self, grads, lrs, active=None, guards=()):
        """grads: flat fp32 CUDA buffer of the same layout; lrs: name -> lr or
        schedule-key -> lr.  active: optional set of array names stepped this
        iteration (the others keep parameters, moments and step counts,
        training.py:513-531); default all.  guards: device status blocks of
        this iteration's renders -- if any of them holds an error the whole
        step is skipped on device (fs4d_status_merge).  The status block is
        reset every step; stream-ordered, check() reads it."""
        lib = N.load()
        self.status.reset()
        for g in guards:
            N.check(lib.fs4d_status_merge(_p(g), _p(self.status.t), 1, _stream()))
        mask = None
        for i, name in enumerate(self.names):
            if active is not None and name not in active:
                continue
            lr = lrs[name] if name in lrs else lrs[schedule_key(name)]
            self.segs[i].lr = float(lr)
        if active is not None:
            mask = (ctypes.c_int32 * max(len(self.names), 1))(*[int(n in active) for n in self.names])
        N.check(lib.fs4d_adam_step_masked(_p(self.params), _p(grads), _p(self.m), _p(self.v), _p(self.steps),
                                          self.segs, mask, len(self.names), _p(self.status.t), _stream()))

    def check(self, st=None):
        """Raise if the last step did not apply: NumericalError
        (numerics.py:149-153) for a non-finite gradient, or the gated render
        error (capacity / numeric) that made it skip.  `st`: an already
        read-back status block."""
        st = self.status.read() if st is None else st
        if int(st[N.ST_CODE]) != 0:
            seg = int(st[N.ST_ADAM_BAD_SEG])
            if seg == N.ADAM_GATED:
                N.raise_device_status(st)
            name, shape = self.specs[seg] if 0 <= seg < len(self.specs) else ("?", ())
            raise NumericalError(f"param {name}: non-finite gradient ({int(st[N.ST_ADAM_BAD_COUNT])} entries) "
                                 f"for param of shape {shape}")
