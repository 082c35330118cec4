"""Multi-process (world_size 2, gloo, CPU) coverage of the N>1 host logic:
timestep sharding for sequence rendering and the flat-gradient all-reduce of
the data-parallel training step (paper_2503_06161_b200/parallel.py)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2503_06161_b200.parallel import (FlatGrads, gradient_specs, sequence_timesteps, shard_range,
                                            shard_timesteps)


def test_shard_range_covers_sequence_contiguously():
    for n, world in [(156, 1), (156, 2), (156, 4), (156, 8), (7, 3), (3, 8), (0, 2)]:
        spans = [shard_range(n, world, r) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == n
        for (a, b), (c, d) in zip(spans, spans[1:]):
            assert b == c
        sizes = [b - a for a, b in spans]
        assert max(sizes) - min(sizes) <= 1
    assert [b - a for a, b in (shard_range(156, 8, r) for r in range(8))] == [20, 20, 20, 20, 19, 19, 19, 19]


def test_shard_timesteps_match_configs2():
    ts = sequence_timesteps(156)
    assert ts[0] == 0.0 and ts[-1] == 1.0 and np.allclose(np.diff(ts), 1 / 155)
    got = np.concatenate([shard_timesteps(156, 4, r) for r in range(4)])
    np.testing.assert_array_equal(got, ts)


def test_gradient_layout_order_and_size():
    specs = gradient_specs(200_000, 16, 3, [[(64, 64, 32)] * 6, [(128, 128, 32)] * 6], [("net.trunk.0.weight", (64, 64))])
    names = [n for n, _ in specs]
    assert names[:7] == ["positions", "rotations", "log_scales", "opacity_logits", "colors_raw", "sh_rest",
                         "features"]
    per_g = sum(int(np.prod(s)) for n, s in specs[:7]) // 200_000
    assert per_g == 75  # K*75 per-Gaussian floats
    fg = FlatGrads(specs, device="cpu")
    fg["sh_rest"][3, 2, 1] = 5.0
    assert fg.buffer[fg.buffer.nonzero()].item() == 5.0


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        specs = [("positions", (5, 3)), ("grid.l0.p0", (4, 4, 2)), ("net.trunk.0.weight", (3, 2))]
        fg = FlatGrads(specs, device="cpu")
        # each rank contributes its own per-pair gradients with the 1/(pairs*world) weight folded in
        for name, _ in specs:
            fg[name].copy_(torch.full(fg[name].shape, float(rank + 1)) / world)
        fg.allreduce_sum()
        # the two-bucket exchange of TrainStep (pass-through rows async, the
        # rest after): the same sums as one all-reduce of the whole buffer
        specs = gradient_specs(5, 4, 1, [[(3, 2, 2)] * 6], [("net.trunk.0.weight", (3, 2))])
        fg = FlatGrads(specs, device="cpu")
        for name, _ in specs:
            fg[name].copy_(torch.full(fg[name].shape, float(rank + 1)) / world)
        fg.allreduce_sum()
        fb = FlatGrads(specs, device="cpu")
        for name, _ in specs:
            fb[name].copy_(torch.full(fb[name].shape, float(rank + 1)) / world)
        lo, hi = fb.span("rotations", "features")
        assert 0 < lo < hi < fb.numel
        work = fb.allreduce_sum_range(lo, hi, async_op=True)
        fb.allreduce_sum_range(0, lo)
        fb.allreduce_sum_range(hi, fb.numel)
        work.wait()
        assert torch.equal(fb.buffer, fg.buffer)
        ts = shard_timesteps(156, world, rank)
        q.put((rank, {n: fg[n].clone().numpy() for n, _ in specs}, ts.tolist()))
    finally:
        dist.destroy_process_group()


def test_flat_grad_allreduce_world2_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda r: r[0])
    for _, grads, _ in res:
        for v in grads.values():
            np.testing.assert_allclose(v, (1 + 2) / 2.0)   # mean of the two ranks' contributions
    all_ts = res[0][2] + res[1][2]
    np.testing.assert_allclose(all_ts, sequence_timesteps(156))


def _bench_worker(rank, world, port, q):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        import bench
        # every rank times its own frames; the job time is the slowest rank's
        ms = bench.dist_max(10.0 + 5.0 * rank, world)
        bench.barrier(world)
        lo, hi = shard_range(156, world, rank)
        q.put((rank, ms, hi - lo))
    finally:
        dist.destroy_process_group()


def test_bench_max_over_ranks_world2_gloo():
    """bench.py's N>1 plumbing: the timed region is the max over ranks and the
    156 configs[2] timesteps split 78 / 78."""
    world = 2
    port = 29500 + (os.getpid() % 1000) + 7
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_bench_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert [r[1] for r in res] == [15.0, 15.0]
    assert sum(r[2] for r in res) == 156 and res[0][2] == 78
