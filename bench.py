"""Benchmark: RGB+feature frames/s of the FE-4DGS per-frame render path
(deform at time t + tile rasterizer) on BASELINE.json configs[1]
(200k Gaussians, 640x512, fx=fy=560, SH3, D=16, HexPlane (1,2)x(64,64,64,25)x32,
MLP width 64 depth 1, Xavier weights, planes U[0.1,0.5]).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one frame (fs4d_deform_fwd + fs4d_render_fwd) at a fresh t on every
rank; ranks render disjoint timesteps (configs[2]'s frame sharding: weak
scaling, no data-path collective).  Inputs are seeded synthetic stand-ins for
EndoNeRF (no dataset access).  `--impl reference` times the reference
algorithm's CPU implementation (the float64 oracle port in oracle/, since the
Python reference cannot travel to the GPU box) on bounded samples of the same
workload with all host cores.
"""

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

K_GAUSS, H, W, FOCAL, SH_DEG, D = 200_000, 512, 640, 560.0, 3, 16
WORKLOAD = "configs[1]: EndoNeRF-shaped frame, 200k Gaussians, 640x512, fx=fy=560, SH3, D=16"
METRIC = "RGB+feature frames/s per B200 at 640x512, 200k Gaussians, D=16; 1/2/4/8 GPU"
PUBLISHED_FPS = None  # paper's 287.95 FPS is RTX 5090 / D=128 -> not the same metric


def f32(x):
    return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)


def make_scene(seed=0, k=K_GAUSS, h=H, w=W, focal=FOCAL, d=D):
    """Seeded configs[1] scene; the arguments give the other
    configs the same distributions (configs[0] size: k=10_000, 128x160, f=150)."""
    import paper_2503_06161_b200 as fs
    rng = np.random.default_rng(seed)
    q = rng.normal(size=(k, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    sh = rng.normal(0.0, 0.2, size=(k, 16, 3))
    cloud = fs.GaussianCloud(
        positions=f32(np.column_stack([rng.uniform(-1, 1, k), rng.uniform(-1, 1, k), rng.uniform(3, 6, k)])),
        rotations=f32(q), log_scales=f32(rng.normal(-4.0, 0.5, size=(k, 3))),
        opacity_logits=f32(rng.normal(0.0, 1.0, size=k)),
        colors_raw=f32(sh[:, 0, :]), features=f32(rng.normal(size=(k, d))), sh_rest=f32(sh[:, 1:, :]))
    field = fs.HexPlaneField(fs.HexPlaneConfig(levels=(1, 2), base_resolution=(64, 64, 64, 25), out_dim=64),
                             fs.scene_aabb(cloud), rng, init="uniform")
    for level in field.planes:
        for i in range(6):
            level[i] = f32(level[i])
    net = fs.DeformationNet(64, fs.DeformationConfig(width=64, depth=1, feature_dim=d), rng, init="xavier",
                            head_init="xavier")
    for _, st in net.stacks():
        for layer in st:
            layer.weight = f32(layer.weight)
    Kmat = np.array([[focal, 0, (w - 1) / 2], [0, focal, (h - 1) / 2], [0, 0, 1.0]])
    return cloud, field, net, Kmat


# ---------------------------------------------------------------------------
# algorithmic work
# ---------------------------------------------------------------------------
def plane_floats():
    res = {1: (64, 64, 64, 25), 2: (128, 128, 128, 25)}
    axes = ((0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3))
    return sum(res[m][a] * res[m][b] * 32 for m in (1, 2) for a, b in axes)


MLP_PARAMS = 64 * 64 + 64 + 4 * (64 * 32 + 32 + 32 * 32 + 32) + (32 * 3 + 3 + 32 * 4 + 4 + 32 * 3 + 3 + 32 + 1) \
    + 128 * 32 + 32 + 32 * D + D
FRAME_BYTES = K_GAUSS * 4 * (11 + D + 3 * (SH_DEG + 1) ** 2) + 4 * plane_floats() + 4 * MLP_PARAMS \
    + H * W * 4 * (3 + D + 1 + 1)
MLP_FLOPS = 2 * 21344 * K_GAUSS
# FP32 work of one evaluated (pixel, Gaussian) in the blend, following the
# reference's per-entry arithmetic (rasterizer.py:215-261): offset 2, power
# 8 (4 mul + 2 fma), opacity x exp 1, w = alpha T 1, 20 accumulated channels
# (RGB, depth, D = 16 features) x 2, transmittance update 2; the exp2 runs on
# the SFU and is not counted.  Evaluations per frame = sum of n_contrib.
BLEND_FLOPS_PER_EVAL = 2 + 8 + 1 + 1 + 2 * (3 + 1 + D) + 2


# stage (library profiler id) -> the single kernel it times (traffic lookup)
STAGE_KERNEL = {"deform_gather": "k_hexplane_latent_c32t", "deform_mlp": "k_mlp_tc_2s", "preprocess": "k_preprocess",
                "blend": "k_blend"}
# per-kernel DRAM traffic + SM utilisation of one `ncu --set full` launch of
# the current kernels (tools/ncu_traffic.py), the newest round's file first
TRAFFIC_JSON = next((f for f in (os.path.join(ROOT, "profiles", n) for n in ("r2_traffic.json", "r1_traffic.json"))
                     if os.path.exists(f)), os.path.join(ROOT, "profiles", "r2_traffic.json"))


def stage_bytes(stage, n_visible, n_pairs):
    """Algorithmic HBM bytes of one launch of each stage (inputs read once + outputs written once)."""
    k = K_GAUSS
    if stage == "deform_fwd":   # cloud geometry+features in, snapshot out, planes + MLP once
        return k * 4 * (11 + D) * 2 + 4 * plane_floats() + 4 * MLP_PARAMS
    if stage == "deform_gather":  # positions in, planes once, latent [K, 64] out
        return k * 4 * 3 + 4 * plane_floats() + k * 4 * 64
    if stage == "deform_mlp":   # latent + cloud geometry/features in, snapshot out, MLP once
        return k * 4 * 64 + k * 4 * (11 + D) * 2 + 4 * MLP_PARAMS
    if stage == "preprocess":   # snapshot (incl. SH) in, 96 B projected record out
        return k * 4 * (11 + D + 3 * (SH_DEG + 1) ** 2) + n_visible * 96
    if stage == "blend":        # projected records + features of the visible set, image out
        return n_visible * (8 + 16 + 16 + 16 + 4 * D) + n_pairs * 4 + H * W * 4 * (3 + 1 + D + 1)
    if stage == "depth_sort":   # key+value in/out once
        return k * 16
    if stage == "binning":      # pairs written once (key+value), ranges
        return n_pairs * 8 + k * 16
    return 0


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


# ---------------------------------------------------------------------------
# clocks sampling (B200_PROFILING.md clocks line)
# ---------------------------------------------------------------------------
class ClockSampler:
    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None
        self.th = None

    def __enter__(self):
        self.stop = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.handle = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.handle, pynvml.NVML_CLOCK_SM)
            self.th = threading.Thread(target=self._poll, daemon=True)
            self.th.start()
            return self
        except Exception:
            self.nv = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}",
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def _poll(self):
        nv = self.nv
        bits = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
                "sw_power_cap": 0x4}
        while not self.stop:
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.handle, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.handle)
                act = ["active" if rs & b else "not active" for b in bits.values()]
                self.rows.append([str(sm), str(self.max_mhz), hex(rs)] + act)
            except Exception:
                pass
            time.sleep(0.002)

    def __exit__(self, *a):
        self.stop = True
        if self.th is not None and self.nv is not None:
            self.th.join(timeout=1)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm = [float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            for n, v in zip(names, r[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# distributed helpers
# ---------------------------------------------------------------------------
def torchrun_command(argv, n_gpus, port):
    """The command bench.py re-executes itself under when asked for N > 1
    GPUs without a torchrun environment: one rank per GPU on this node,
    rendezvous on 127.0.0.1."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={int(n_gpus)}",
            "--master-addr", "127.0.0.1", f"--master-port={int(port)}", os.path.abspath(__file__)] + list(argv)


def _free_port():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def dist_setup(n_gpus):
    """(rank, world, local rank).  Under torchrun the world comes from the
    environment and must equal --gpus; NCCL over NVLink/NVSwitch carries the
    barrier, the max-over-ranks timing and the training all-reduce."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != int(n_gpus):
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {n_gpus}")
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def comm_info(world):
    """The collective backend the ranks actually run (the 'NCCL nranks' line)."""
    if world == 1:
        return {"backend": None, "nranks": 1}
    import torch
    import torch.distributed as dist
    info = {"backend": dist.get_backend(), "nranks": dist.get_world_size()}
    try:
        v = torch.cuda.nccl.version()
        info["nccl_version"] = ".".join(str(x) for x in v) if isinstance(v, tuple) else str(v)
    except Exception:
        pass
    return info


def dist_gather(x, world):
    """Per-rank scalars gathered to every rank (list in rank order)."""
    if world == 1:
        return [x]
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    out = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(out, t)
    return [float(o.item()) for o in out]


def dist_max(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"  # gloo in the CPU tests
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# ---------------------------------------------------------------------------
# CPU baseline: the unmodified reference (featsplat, pip-installed into
# baseline/_ref), whole frames
# ---------------------------------------------------------------------------
REF_PATH = os.path.join(ROOT, "baseline", "_ref")


def load_featsplat():
    """The reference package itself, or None when baseline/_ref is absent."""
    if os.path.isdir(REF_PATH) and REF_PATH not in sys.path:
        sys.path.insert(0, REF_PATH)
    try:
        import featsplat.deformation  # noqa: F401
        import featsplat.rasterizer  # noqa: F401
        import featsplat
        return featsplat
    except Exception:
        return None


def reference_scene(seed=0, k=K_GAUSS, h=H, w=W, focal=FOCAL, d=D):
    """make_scene's configs[1] scene as the reference's own objects.  The
    reference has no SH: its colour is the degree-0 term
    (colors_raw), which is what it renders."""
    import featsplat.deformation as RD
    import featsplat.gaussians as RG
    import featsplat.hexplane as RH
    import featsplat.rasterizer as RR
    cloud, field, net, Kmat = make_scene(seed, k=k, h=h, w=w, focal=focal, d=d)
    rc = RG.GaussianCloud(**{f: np.array(getattr(cloud, f)) for f in
                             ("positions", "rotations", "log_scales", "opacity_logits", "colors_raw", "features")})
    rf = RH.HexPlaneField(RH.HexPlaneConfig(levels=(1, 2), base_resolution=(64, 64, 64, 25), out_dim=64), field.aabb,
                          np.random.default_rng(1))
    rf.planes = [[np.array(p) for p in lv] for lv in field.planes]
    rn = RD.DeformationNet(64, RD.DeformationConfig(width=64, depth=1, feature_dim=d), np.random.default_rng(2))
    for (_, st), (_, st2) in zip(rn.stacks(), net.stacks()):
        for layer, src in zip(st, st2):
            layer.weight, layer.bias = np.array(src.weight), np.array(src.bias)
    frame = RG.CameraFrame(K=Kmat, T=np.eye(4), time=0.0, image=np.zeros((h, w, 3)), depth=np.zeros((h, w)),
                           mask=np.ones((h, w), dtype=bool))
    return rc, rf, rn, frame, RR.RasterConfig()


def _ref_init():
    # one BLAS thread per worker: the workers are the parallelism
    from threadpoolctl import threadpool_limits
    threadpool_limits(1)


def _ref_frame(t):
    """One whole reference frame in a worker: deformation.deform +
    rasterizer.render (cli.py:58-61) on the fork-inherited scene."""
    S = sys.modules["fs4d_ref_state"]
    t0 = time.perf_counter()
    if S.kind == "reference":
        import featsplat.deformation as RD
        import featsplat.rasterizer as RR
        snap = RD.deform(S.cloud, S.field, S.net, float(t))
        RR.render(snap, S.frame, S.cfg)
    else:  # oracle port (baseline/_ref absent)
        from oracle import fs4d_oracle as O
        snap, _ = O.deform(S.cloud, S.field.planes, S.field.aabb, S.net, float(t))
        snap = type("C", (), dict(snap, sh_rest=getattr(S.cloud, "sh_rest", None)))()
        O.render(snap, S.K, np.eye(4), H, W, O.RasterParams())
    return time.perf_counter() - t0


def host_info():
    ncores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    avail = None
    try:
        with open("/proc/meminfo") as fh:
            for line in fh:
                if line.startswith("MemAvailable:"):
                    avail = int(line.split()[1]) * 1024
    except Exception:
        pass
    if avail is None:
        avail = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
    return {"cpu_count": os.cpu_count(), "affinity": ncores, "mem_available_gb": round(avail / 2 ** 30, 1)}


REF_FRAME_GB = 16.0  # peak RSS of one configs[1] reference frame (~15 GB)


def cpu_reference(timed_frames, warm_frames, seed=0, procs=None):
    """Whole configs[1] frames of the reference CPU path, P worker processes
    (one frame each, one BLAS thread each) over the host cores; returns the
    aggregate frames/s of the timed frames."""
    import multiprocessing as mp
    import types
    fsp = load_featsplat()
    mod = types.ModuleType("fs4d_ref_state")
    if fsp is not None:
        mod.kind = "reference"
        mod.cloud, mod.field, mod.net, mod.frame, mod.cfg = reference_scene(seed)
    else:
        mod.kind = "port"
        cloud, field, net, Kmat = make_scene(seed)
        mod.cloud, mod.field, mod.K = cloud, field, Kmat
        mod.net = {p: [(l.weight, l.bias, l.activation == "relu") for l in st] for p, st in net.stacks()}
    sys.modules["fs4d_ref_state"] = mod
    info = host_info()
    cap = max(1, int(info["mem_available_gb"] // REF_FRAME_GB))
    procs = procs or max(1, min(info["affinity"], cap, max(timed_frames, 1)))
    ts = np.arange(156) / 155.0
    ctx = mp.get_context("fork")
    with ctx.Pool(procs, initializer=_ref_init) as pool:
        if warm_frames:
            pool.map(_ref_frame, [ts[i % 156] for i in range(warm_frames)], chunksize=1)
        t0 = time.perf_counter()
        per = pool.map(_ref_frame, [ts[(warm_frames + i) % 156] for i in range(timed_frames)], chunksize=1)
        wall = time.perf_counter() - t0
    desc = ("unmodified featsplat 0.1.0 (baseline/_ref): deformation.deform + rasterizer.render, SH degree 0 "
            "(the reference has no SH)" if mod.kind == "reference" else "oracle/fs4d_oracle.py float64 port")
    return {"value": timed_frames / wall, "cores": procs, "kind": mod.kind, "host": info,
            "frame_s_mean": float(np.mean(per)), "frame_s_max": float(np.max(per)), "wall_s": wall,
            "sample": f"{timed_frames} whole configs[1] frames (t = k/155) of the {desc}, {procs} worker processes "
                      f"x 1 BLAS thread, value = frames / wall time; mean {np.mean(per):.1f} s per frame per "
                      f"process"}


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def gpu_bench(args, rank, world, local):
    import torch
    import paper_2503_06161_b200 as fs
    from paper_2503_06161_b200 import device as dv

    torch.cuda.set_device(local)
    cloud_np, field_np, net_np, Kmat = make_scene(0)
    cloud = dv.DeviceCloud.from_cloud(cloud_np)
    field = dv.DeviceField.from_field(field_np)
    if os.environ.get("FS4D_LOCALITY", "1") == "1":
        # Morton visiting order of the canonical positions for the HexPlane
        # gather: a property of the model, computed once (untimed) like any
        # index; results are bit-identical in any order (tested).  Measured
        # +2.5% frames/s (gather 72 -> 66 us)
        field = field.with_order(dv.locality_order(cloud.positions, field.aabb))
    net = dv.DeviceNet.from_net(net_np)
    cfg = fs.RasterConfig()
    pipe = dv.FramePipeline(cloud, field, net, H, W, cfg)
    T = np.eye(4)
    # timesteps of configs[2]: t = k/155, sharded contiguously over ranks; cycled for K steps
    ts = np.arange(156) / 155.0
    mine = np.array_split(ts, world)[rank]
    steps, warm = args.steps, args.warmup

    # size the pair buffer once (host-synchronous check), then run fully async
    pipe.run(float(mine[0]), Kmat, T, check=True)
    torch.cuda.synchronize()
    st = pipe.renderer.status.read()
    n_vis = int(st[2])
    n_pairs = (int(st[4]) << 32) | (int(st[3]) & 0xFFFFFFFF)
    n_eval = int(pipe.images["n_contrib"].sum().item())  # evaluated (pixel, Gaussian) entries of one frame
    pipe.renderer.cap = int(n_pairs * 1.5) + 4096
    flush = torch.empty(256 * 2 ** 20 // 4, dtype=torch.float32, device="cuda")  # > 126 MB L2

    for i in range(warm):
        pipe.run(float(mine[i % len(mine)]), Kmat, T)
    torch.cuda.synchronize()

    # serial reference number: one frame at a time, L2 flushed between frames
    stream = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    barrier(world)
    torch.cuda.synchronize()
    for i in range(steps):
        flush.zero_()  # L2 flush between timed iterations (outside the events)
        ev[i][0].record(stream)
        pipe.run(float(mine[i % len(mine)]), Kmat, T)
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    barrier(world)
    ms_serial = dist_max(sum(a.elapsed_time(b) for a, b in ev), world)
    st = pipe.renderer.status.read()
    if int(st[0]) != 0:
        raise RuntimeError(f"device status {st[:5]} during timed region")

    # headline: the configs[2] sequence with three frames in flight on three
    # streams over six model replicas (6 x 70 MB rotate through far more than
    # the 126 MB L2, so no flush is needed between frames); each step = one frame
    n_str = int(os.environ.get("FS4D_SEQ_STREAMS", "3"))  # A/B knob; replicas = 2 x streams
    seq = dv.SequenceRenderer(cloud, field, net, H, W, cfg, pipelines=2 * n_str, streams=n_str, replicas=2 * n_str)
    seq.warm(float(mine[0]), Kmat, T, pair_capacity=pipe.renderer.cap)
    ts_seq = [float(mine[i % len(mine)]) for i in range(steps)]
    seq.run([float(mine[i % len(mine)]) for i in range(warm)], Kmat, T)
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        a_ev, b_ev = seq.run(ts_seq, Kmat, T)
        torch.cuda.synchronize()
    barrier(world)
    ms_rank = a_ev.elapsed_time(b_ev)
    ms_max = dist_max(ms_rank, world)
    per_rank_ms = dist_gather(ms_rank, world)
    seq.raise_if_error()

    # per-stage timing pass (events around each stage on the launching stream)
    dv.profile_collect()
    dv.profile_enable(True)
    for i in range(steps):
        flush.zero_()
        pipe.run(float(mine[i % len(mine)]), Kmat, T)
    torch.cuda.synchronize()
    prof = dv.profile_collect()
    dv.profile_enable(False)

    # end-to-end through the public API with host buffers: every frame copies
    # the whole canonical cloud (60 MB) host->device from pinned memory and
    # the colour/depth/feature/alpha images (27.5 MB) back; two pipeline
    # replicas on two streams overlap the copies of neighbouring frames
    sf = dv.StreamedFrames(cloud, field, net, H, W, cfg)
    sf.warm(float(mine[0]), Kmat, T)
    for p in sf.pipes:
        p.renderer.cap = pipe.renderer.cap
    sf.warm(float(mine[0]), Kmat, T)
    ts_e2e = [float(mine[i % len(mine)]) for i in range(steps)]
    sf.run(ts_e2e[:warm], Kmat, T)
    torch.cuda.synchronize()
    barrier(world)
    a, b = sf.run(ts_e2e, Kmat, T)
    torch.cuda.synchronize()
    e2e_ms = dist_max(a.elapsed_time(b), world)
    for p in sf.pipes:
        st = p.renderer.status.read()
        if int(st[0]) != 0:
            raise RuntimeError(f"device status {st[:5]} during the e2e region")
    return dict(ms=ms_max, ms_serial=ms_serial, prof=prof, clocks=clk.summary(), n_vis=n_vis, n_pairs=n_pairs,
                e2e_ms=e2e_ms, n_eval=n_eval, h2d=sf.h2d_bytes(), d2h=sf.d2h_bytes(), steps=steps, per_rank_ms=per_rank_ms,
                comm=comm_info(world))


def train_bench(args, rank, world, local):
    """configs[4]: 8 (view, t) pairs per GPU, L1 RGB + L1 feature, backward
    through rasterizer and deformation, one flat-gradient all-reduce."""
    import torch
    import paper_2503_06161_b200 as fs
    from paper_2503_06161_b200 import device as dv
    from paper_2503_06161_b200.train import TrainStep

    torch.cuda.set_device(local)
    cloud_np, field_np, net_np, Kmat = make_scene(0)
    fine = args.workload == "fine"
    gen = torch.Generator(device="cuda")
    gen.manual_seed(rank)
    if fine:
        # the reference's fine-stage iteration (training.py:489-535) with its
        # TrainConfig defaults (training.py:53-83): masked RGB L1 + depth L1,
        # pointwise decoder against a 16-channel teacher at 1/4 resolution,
        # HexPlane TV, then Adam on every parameter array
        from paper_2503_06161_b200.numerics import LrSchedule
        ct = 16
        dec_w = (torch.rand(ct, D, device="cuda", generator=gen) * 2 - 1) * float(np.sqrt(6.0 / D))
        dec = (dec_w, torch.zeros(ct, device="cuda"))
        step = TrainStep(dv.DeviceCloud.from_cloud(cloud_np), dv.DeviceField.from_field(field_np),
                         dv.DeviceNet.from_net(net_np), H, W, fs.RasterConfig(), world=world, loss_mode="decoder",
                         lambda_rgb=1.0, lambda_depth=0.01, lambda_feat=1.0, lambda_tv=0.03, decoder=dec)
        step.attach_optimizer({
            "positions": LrSchedule(1.6e-4, 1.6e-6, 7000), "rotations": LrSchedule.constant(1e-3),
            "log_scales": LrSchedule.constant(5e-3), "opacity_logits": LrSchedule.constant(5e-2),
            "colors_raw": LrSchedule.constant(2.5e-3), "features": LrSchedule.constant(2.5e-3),
            "grid": LrSchedule(3.2e-3, 3.2e-6, 7000), "net": LrSchedule(1.6e-4, 1.6e-7, 7000, 0.01, 0),
            "decoder": LrSchedule.constant(1e-3)})
    else:
        step = TrainStep(dv.DeviceCloud.from_cloud(cloud_np), dv.DeviceField.from_field(field_np),
                         dv.DeviceNet.from_net(net_np), H, W, fs.RasterConfig(), world=world)
    rng = np.random.default_rng(100 + rank)
    pairs = 8

    def rigid():
        axis = rng.normal(size=3)
        axis /= np.linalg.norm(axis)
        ang = np.deg2rad(rng.uniform(-5, 5))
        Kx = np.array([[0, -axis[2], axis[1]], [axis[2], 0, -axis[0]], [-axis[1], axis[0], 0]])
        T = np.eye(4)
        T[:3, :3] = np.eye(3) + np.sin(ang) * Kx + (1 - np.cos(ang)) * Kx @ Kx
        T[:3, 3] = rng.uniform(-0.1, 0.1, 3)
        return T

    if fine:
        batch = [(float(rng.uniform()), Kmat, rigid(),
                  torch.rand(H, W, 3, device="cuda", generator=gen),
                  torch.randn(H // 4, W // 4, 16, device="cuda", generator=gen),
                  (torch.rand(H, W, device="cuda", generator=gen) > 0.05).to(torch.uint8),
                  torch.rand(H, W, device="cuda", generator=gen) * 3 + 3) for _ in range(pairs)]
    else:
        batch = [(float(rng.uniform()), Kmat, rigid(),
                  torch.rand(H, W, 3, device="cuda", generator=gen),
                  torch.randn(H, W, D, device="cuda", generator=gen)) for _ in range(pairs)]
    step.run(batch, check=True)  # sizes the pair buffer
    for _ in range(args.warmup):
        step.run(batch)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(world)
    torch.cuda.synchronize()
    a.record(stream)
    for _ in range(args.steps):
        step.run(batch)
    b.record(stream)
    torch.cuda.synchronize()
    ms = dist_max(a.elapsed_time(b), world)
    per_rank_ms = dist_gather(a.elapsed_time(b), world)
    # per-stage times from one serial step (one lane: with pairs in flight the
    # stage events of concurrent streams would overlap)
    lanes = step.n_lanes
    step.n_lanes, step._lanes = 1, None
    step.run(batch)
    torch.cuda.synchronize()
    dv.profile_collect()
    dv.profile_enable(True)
    step.run(batch)
    torch.cuda.synchronize()
    prof = dv.profile_collect()
    dv.profile_enable(False)
    step.n_lanes, step._lanes = lanes, None
    return dict(ms=ms, prof=prof, loss=float(step.loss.item()), grad_floats=step.grads.numel, pairs=pairs,
                lanes=lanes, per_rank_ms=per_rank_ms, comm=comm_info(world))


def blend_fp32(r, stage_ms):
    import torch
    if not stage_ms.get("blend"):
        return None
    prop = torch.cuda.get_device_properties(0)
    mhz = (r["clocks"] or {}).get("sm_max_mhz") or 1965.0
    peak = prop.multi_processor_count * 128 * 2 * mhz * 1e6 / 1e12
    flops = r["n_eval"] * BLEND_FLOPS_PER_EVAL
    ach = flops / (stage_ms["blend"] / 1000.0) / 1e12
    return {"bound": "fp32", "kernel": "k_blend", "achieved": ach, "peak": peak, "unit": "TFLOP/s",
            "frac": ach / peak, "evals_per_frame": r["n_eval"], "flops_per_eval": BLEND_FLOPS_PER_EVAL,
            "peak_source": f"{prop.multi_processor_count} SMs x 128 x 2 x {mhz:.0f} MHz"}


def launches_per_frame():
    """libfs4d kernels per frame: deform (pack, HexPlane latent, tcgen05 MLP) and
    render (status reset, preprocess + fused tile histogram, pair partition
    with the fused tile-offset scan, per-tile sort, blend)."""
    return 3 + (1 + 1 + 1 + 1 + 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--workload", default="render", choices=["render", "train", "fine"])
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-execute under torchrun (the driver launches
        # it that way itself; this makes `python bench.py --gpus N` equivalent)
        sys.exit(subprocess.call(torchrun_command(sys.argv[1:], args.gpus, _free_port())))

    rank, world, local = dist_setup(args.gpus)
    base = {"metric": METRIC, "unit": "frames/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded stand-in for EndoNeRF, SURVEY §8(d); z~U[3,6])",
            # identical in both arms (the driver compares them); each arm's
            # execution details go under "setup"
            "config": {"workload": WORKLOAD, "frames_per_rank_step": 1, "timesteps": "t=k/155 sharded by rank",
                       "parallelism": f"frame-sharded x{world}"}}

    if args.impl == "reference":
        if rank != 0:
            return
        r = cpu_reference(args.steps, args.warmup)
        line = dict(base)
        line.update({"impl": "reference", "value": r["value"], "ms_per_step": 1000.0 / r["value"],
                     "n_gpus": world, "setup": {"cpu": "whole frames, one per worker process (see cpu_baseline)"},
                     "cpu_baseline": {"value": r["value"], "unit": "frames/s", "cores": r["cores"],
                                      "kind": r["kind"], "sample": r["sample"]},
                     "host": r["host"],
                     "e2e": {"value": r["value"], "unit": "frames/s", "h2d_bytes_per_step": 0,
                             "d2h_bytes_per_step": 0}})
        print(json.dumps(line))
        return

    if args.workload in ("train", "fine"):
        r = train_bench(args, rank, world, local)
        if rank == 0:
            line = dict(base)
            metric = "configs[4] training steps/s (8 (view,t) pairs per GPU, fwd+bwd+allreduce)"
            if args.workload == "fine":
                metric = ("fine-stage training steps/s (configs[4] scene, 8 pairs/GPU, masked RGB+depth L1, decoder "
                          "feature loss, TV, all-reduce, Adam)")
            line.update({"metric": metric,
                         "unit": "steps/s", "value": world * args.steps / (r["ms"] / 1000.0) / world,
                         "ms_per_step": r["ms"] / args.steps,
                         "frames_per_s": world * r["pairs"] * args.steps / (r["ms"] / 1000.0),
                         "stage_ms_per_step": {s: round(ms, 4) for s, (ms, c) in r["prof"].items() if c},
                         "allreduce_floats": r["grad_floats"], "loss": r["loss"], "comm": r["comm"],
                         "per_rank_steps_per_s": [args.steps / (m / 1000.0) for m in r["per_rank_ms"]]})
            line["config"] = dict(base["config"], workload="configs[4]: configs[1] scene, 8 (view,t) pairs/GPU, "
                                                           "L1 RGB + L1 feature", parallelism=f"dp{world}",
                                  pairs_in_flight=r["lanes"], stage_ms="one serial (1-lane) step")
            line["setup"] = {"l2": "flushed (256 MB write) between steps"}
            if args.workload == "fine":
                line["config"]["workload"] = ("reference fine-stage iteration (training.py:489-535) on the configs[1] "
                                              "scene: 8 pairs/GPU, teacher 16ch at 160x128, TrainConfig defaults")
            print(json.dumps(line))
        return
    r = gpu_bench(args, rank, world, local)
    ns = int(os.environ.get("FS4D_SEQ_STREAMS", "3"))
    base["setup"] = {"gather_order": ("morton (once per model, untimed; bit-identical results)"
                                      if os.environ.get("FS4D_LOCALITY", "1") == "1" else "source"),
                     "frames_in_flight": f"{ns} per GPU ({ns} streams)",
                     "l2": f"no flush: {2 * ns} rotating model replicas ({2 * ns} x 70 MB > 126 MB L2); "
                           "value_serial is flushed (256 MB write) between frames"}
    hbm, tf, peak_src = peaks()
    frames = world * r["steps"]
    value = frames / (r["ms"] / 1000.0)
    prof = r["prof"]
    stage_ms = {s: (ms / c if c else 0.0) for s, (ms, c) in prof.items()}
    fwd = {s: v for s, v in stage_ms.items() if s in ("deform_fwd", "preprocess", "depth_sort", "binning", "blend")}
    frame_ms = sum(fwd.values())
    # dominant single kernel (binning is a chain of small kernels, excluded)
    single = {s: stage_ms[s] for s in STAGE_KERNEL if stage_ms.get(s)}
    top = max(single, key=single.get)
    top_bytes = stage_bytes(top, r["n_vis"], r["n_pairs"])
    achieved = top_bytes / (stage_ms[top] / 1000.0) / 1e9
    traffic, traffic_src, utilisation = None, None, None
    try:
        with open(TRAFFIC_JSON) as fh:
            t = json.load(fh)[STAGE_KERNEL[top]]
        traffic = t["dram_read_bytes"] + t["dram_write_bytes"]
        traffic_src = f"{os.path.basename(TRAFFIC_JSON)}: ncu --set full of {t['kernel'].split('(')[0]} (one launch)"
        utilisation = t.get("utilisation")
    except Exception:
        utilisation = None
    kernels = {s: {"ms": round(stage_ms[s], 4), "algorithmic_bytes": stage_bytes(s, r["n_vis"], r["n_pairs"]),
                   "achieved_gbs": stage_bytes(s, r["n_vis"], r["n_pairs"]) / (stage_ms[s] / 1000.0) / 1e9}
               for s in single}
    line = dict(base)
    line.update({
        "value": value, "ms_per_step": r["ms"] / r["steps"],
        "value_serial": {"value": frames / (r["ms_serial"] / 1000.0), "ms_per_frame": r["ms_serial"] / r["steps"],
                         "note": "one frame at a time on one stream, 256 MB L2 flush between frames"},
        "roofline": {"bound": "hbm", "kernel": STAGE_KERNEL[top], "stage": top, "achieved": achieved, "peak": hbm,
                     "unit": "GB/s", "frac": achieved / hbm, "traffic": traffic, "traffic_source": traffic_src,
                     "peak_source": peak_src, "algorithmic_bytes_per_launch": top_bytes,
                     "share_of_step": stage_ms[top] / frame_ms if frame_ms else None,
                     # the kernel is issue/latency bound, not HBM bound: SM-side utilisation of the
                     # same ncu capture (percent of B200 peak)
                     "sm_utilisation_pct": utilisation},
        "kernels": kernels,
        # secondary roofline: the blend is FP32-issue bound; peak =
        # SMs x 128 FP32 lanes x 2 (FMA) x the max SM clock
        "roofline_fp32": blend_fp32(r, stage_ms),
        "roofline_frame": {"bytes_per_frame": FRAME_BYTES,
                           "achieved_gbs": FRAME_BYTES / (r["ms"] / r["steps"] / 1000.0) / 1e9,
                           "frac": FRAME_BYTES / (r["ms"] / r["steps"] / 1000.0) / 1e9 / hbm},
        "stage_ms": {k: round(v, 4) for k, v in stage_ms.items() if v},
        "mlp": {"flops_per_frame": MLP_FLOPS, "kernel": "k_mlp_tc_2s (bf16x3 on tcgen05: 3x these flops issued)",
                "tflops": MLP_FLOPS / (stage_ms["deform_mlp"] / 1000.0) / 1e12 if stage_ms.get("deform_mlp") else None,
                "peak_bf16_tflops": tf, "frac_of_bf16_peak_issued": 3 * MLP_FLOPS / (stage_ms["deform_mlp"] / 1000.0)
                / 1e12 / tf if stage_ms.get("deform_mlp") else None},
        "work": {"visible": r["n_vis"], "pairs": r["n_pairs"]},
        "clocks": r["clocks"],
        "e2e": {"value": frames / (r["e2e_ms"] / 1000.0), "unit": "frames/s", "h2d_bytes_per_step": r["h2d"],
                "d2h_bytes_per_step": r["d2h"],
                # the e2e bound: host link bytes per second (PCIe, both directions overlap)
                "link_gbs": {"h2d": r["h2d"] * frames / (r["e2e_ms"] / 1000.0) / 1e9,
                             "d2h": r["d2h"] * frames / (r["e2e_ms"] / 1000.0) / 1e9}},
        "gpu_launches": launches_per_frame() * r["steps"],
        "per_rank_frames_per_s": [r["steps"] / (m / 1000.0) for m in r["per_rank_ms"]],
        "comm": r["comm"],
    })
    if rank == 0 and world == 1 and not args.no_cpu:
        # bounded sample: one wave of whole reference frames, one per worker process
        c = cpu_reference(max(1, min(host_info()["affinity"], int(host_info()["mem_available_gb"] // REF_FRAME_GB))), 0)
        line["cpu_baseline"] = {"value": c["value"], "unit": "frames/s", "cores": c["cores"], "kind": c["kind"],
                                "sample": c["sample"]}
    if rank == 0:
        print(json.dumps(line))


if __name__ == "__main__":
    main()
