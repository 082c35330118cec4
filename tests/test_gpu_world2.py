"""World-size-2 runs of the multi-GPU paths on ONE GPU: two
processes, torch.distributed over gloo with CUDA tensors, each rank with its
own replica.  The ranks' kernels never wait on one another (the only exchange
is the host-staged gloo all-reduce), so sharing one device is a faithful
stand-in for the data flow, not for NVLink bandwidth.

* Training (configs[4] shape, reduced): each rank runs TrainStep(world=2) on
  its half of 4 (view, t) pairs; the all-reduced flat gradient buffer and
  loss equal a world-1 TrainStep over all 4 pairs (fp32 summation order
  aside), and both ranks hold identical buffers.
* Sequence rendering (configs[2] shape, reduced): each rank renders its
  contiguous shard of the timesteps (parallel.shard_timesteps); the union of
  the shards is bit-identical to a single rank rendering every frame.
"""

import socket

import numpy as np
import pytest

from conftest import has_gpu, pinhole, random_cloud_arrays, rigid_T

pytestmark = pytest.mark.gpu

H, W, D = 48, 64, 8
N_FRAMES = 10


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not has_gpu():
        pytest.skip("no CUDA device")
    import __graft_entry__ as ge
    ge.build()


def _scene():
    import paper_2503_06161_b200 as fs
    rng = np.random.default_rng(77)
    a = random_cloud_arrays(rng, 3000, D, depth_range=(2.0, 4.0), xy=1.0, ls_range=(0.02, 0.1), sh_degree=1)
    cloud = fs.GaussianCloud(**a)
    field = fs.HexPlaneField(fs.HexPlaneConfig(levels=(1, 2), base_resolution=(8, 8, 8, 4), out_dim=64),
                             fs.scene_aabb(cloud), rng, init="uniform")
    net = fs.DeformationNet(64, fs.DeformationConfig(width=64, depth=1, feature_dim=D), rng, init="xavier",
                            head_init="xavier")
    pairs = []
    for t in (0.1, 0.35, 0.6, 0.9):
        pairs.append((t, rigid_T(rng), rng.uniform(size=(H, W, 3)).astype(np.float32),
                      rng.normal(size=(H, W, D)).astype(np.float32)))
    return cloud, field, net, pairs


def _train(pairs, world, group_ranks=None, lanes=1, overlap=False, deterministic=False):
    import torch
    import paper_2503_06161_b200 as fs
    from paper_2503_06161_b200 import device as dv
    from paper_2503_06161_b200.train import TrainStep
    cloud, field, net, _ = _scene()
    step = TrainStep(dv.DeviceCloud.from_cloud(cloud), dv.DeviceField.from_field(field), dv.DeviceNet.from_net(net),
                     H, W, fs.RasterConfig(), world=world, lanes=lanes, deterministic=deterministic)
    step.overlap_allreduce = overlap
    K = pinhole(H, W, 50.0)
    batch = [(t, K, T, torch.as_tensor(tr, device="cuda"), torch.as_tensor(tf, device="cuda"))
             for t, T, tr, tf in pairs]
    loss = float(step.run(batch, check=True).item())
    torch.cuda.synchronize()
    return loss, step.grads.buffer.double().cpu().numpy()


def _frames(ts):
    import torch
    import paper_2503_06161_b200 as fs
    from paper_2503_06161_b200 import device as dv
    cloud, field, net, _ = _scene()
    pipe = dv.FramePipeline(dv.DeviceCloud.from_cloud(cloud), dv.DeviceField.from_field(field),
                            dv.DeviceNet.from_net(net), H, W, fs.RasterConfig())
    out = []
    for t in ts:
        pipe.run(float(t), pinhole(H, W, 50.0), np.eye(4), check=True)
        out.append({k: v.cpu().numpy().copy() for k, v in pipe.images.items()})
    return out


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2503_06161_b200.parallel import shard_range, shard_timesteps
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        _, _, _, pairs = _scene()
        lo, hi = shard_range(len(pairs), world, rank)
        # two lanes per rank: both gradient buckets (pass-through rows on
        # the side stream, the rest after the backward) see a lane sum
        loss, grads = _train(pairs[lo:hi], world, lanes=2)
        frames = _frames(shard_timesteps(N_FRAMES, world, rank))
        q.put((rank, loss, grads, frames))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_world2_training_and_sequence_shards_match_world1():
    import torch.multiprocessing as mp
    from paper_2503_06161_b200.parallel import sequence_timesteps
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=600) for _ in range(world)), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0

    _, _, _, pairs = _scene()
    loss1, grads1 = _train(pairs, 1)
    scale = np.abs(grads1).max()
    for rank, loss, grads, _ in res:
        assert abs(loss - loss1) < 1e-9 * max(1.0, abs(loss1)), (rank, loss, loss1)
        err = np.abs(grads - grads1).max()
        assert err < 1e-5 * scale, (rank, err, scale)
    np.testing.assert_array_equal(res[0][2], res[1][2])  # replicas hold the same reduced buffer

    frames1 = _frames(sequence_timesteps(N_FRAMES))
    sharded = res[0][3] + res[1][3]
    assert len(sharded) == N_FRAMES
    for a, b in zip(sharded, frames1):
        for key in b:
            np.testing.assert_array_equal(a[key], b[key], err_msg=key)


def test_overlapped_allreduce_buckets_bitwise_equal_single_reduce():
    """The two-bucket exchange (pass-through rows summed and reduced on a side
    stream during the backward) performs the same sums in the same order as
    the single post-backward reduce: world 1, three lanes, deterministic
    backward (no float atomics), bitwise equal."""
    _, _, _, pairs = _scene()
    loss_a, grads_a = _train(pairs, 1, lanes=3, overlap=False, deterministic=True)
    loss_b, grads_b = _train(pairs, 1, lanes=3, overlap=True, deterministic=True)
    # (the loss itself is a double-precision atomic sum over blocks: last-bit
    # order effects; the gradients are the bitwise claim)
    assert abs(loss_a - loss_b) <= 1e-12 * abs(loss_a)
    np.testing.assert_array_equal(grads_a, grads_b)
