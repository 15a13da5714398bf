"""Benchmark of the ARTEMIS hot path: full posed frames (LBS warp +
Morton-key octree rebuild + render), one step = one unit of the config's
workload.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl artemis|reference]
                    [--config c2|c0|c1|c4] [--shard frames|tiles|peer]

Default workload (the north star's): the configs[2] asset (~1M leaves,
C = 32) rendered 1024x1024, one full posed frame per step, poses/cameras of
the configs[3] sequence on that asset. Other configs: c0 (configs[0], one
256^2 frame per step), c1 (configs[1]: one pose, 8 views of 512^2 per step,
views sharded over the GPUs, ONE NCCL gather to rank 0), c4 (configs[4]: one
stereo frame, 2 x 1440x1600, per GPU per step).

One process per GPU. With --gpus N > 1 and no torchrun environment the
script re-launches itself under torch.distributed.run (127.0.0.1); under
torchrun the world size must equal --gpus. Rank 0 prints ONE JSON line.

  value       rays/s over the job = rays of the K steps on all ranks / max
              over ranks of the summed CUDA-event time of the K graph-
              replayed steps (inputs resident in HBM; L2 flushed between
              steps)
  e2e         the same metric through the public Python API with host
              buffers: per step host FK, H2D of the pose/camera block, the
              device work, any NCCL gather, and the D2H of the result maps
              into pinned host memory (wall clock, max over ranks)
  e2e_api     (c0/c2, N = 1) the reference's own per-frame call,
              pipeline.timed_render_frame -> fp64 FrameBuffers, as the
              installed reference CLI/service calls it
  roofline    the render kernel: algorithmic bytes per launch / its mean
              eager CUDA-event duration
  cpu_baseline  the reference's CPU path (its compiled kernels from
              oracle/_ref, numpy stages restated in oracle/ref_port.py), full
              frames, rank 0 at N = 1 only
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))

FLUSH_BYTES = 256 << 20  # > 126 MB L2

METRICS = {
    "c2": "rays/s (full warp+rebuild+render frame, ~1M-leaf octree, 1024x1024)",
    "c0": "rays/s (full warp+rebuild+render frame, configs[0], 256x256)",
    "c1": "rays/s (one pose: warp+rebuild + 8 views of 512x512, configs[1])",
    "c4": "rays/s (full warp+rebuild+render stereo frame, ~4M-leaf octree, 2x1440x1600)",
}
WORKLOADS = {
    "c2": ("configs[2] asset (512^3 grid, 4-voxel shell, ~985k canonical voxels, 32-channel SH "
           "deg 2, 24 joints) rendered 1024x1024, one full posed frame per step with the "
           "configs[3] pose/camera sequence"),
    "c0": ("configs[0] (128^3 grid, 3-voxel shell, ~29k voxels, 16-channel SH deg 2, 24 "
           "joints), one full posed 256x256 frame per step"),
    "c1": ("configs[1] (configs[0] asset): one pose per step, warp + rebuild, 8 views of "
           "512x512 at azimuths 45 deg apart, elevation 15 deg"),
    "c4": ("configs[4] (1024^3 grid, 3-voxel shell, ~4M voxels, 32-channel SH deg 2, 32 "
           "joints): one full posed stereo frame (2 eyes 1440x1600, 64 mm baseline) per GPU "
           "per step, random-walk pose sequence"),
}


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="artemis", choices=["artemis", "reference"])
    ap.add_argument("--config", default="c2", choices=["c2", "c0", "c1", "c4"])
    ap.add_argument("--shard", default="frames", choices=["frames", "tiles", "peer"],
                    help="c0/c2 at N>1: frames (weak scaling, no collective), 8x4 screen "
                         "tiles of the same frame (strong scaling, one NCCL gather per frame), "
                         "or tiles stored by the render kernels straight into rank 0's maps "
                         "over NVLink (peer: CUDA IPC mapping, no gather)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-frames", type=int, default=3)
    ap.add_argument("--no-cpu-1thread", action="store_true")
    return ap.parse_args(argv)


# ---------------------------------------------------------------------------
# launch: one process per GPU


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def maybe_spawn(args) -> None:
    """--gpus N > 1 without a torchrun environment: re-launch under
    torch.distributed.run with N ranks and exit with its status."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")  # keep stdout to the one JSON line
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    sys.exit(subprocess.run(cmd, env=env).returncode)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def parallelism(args, world) -> str:
    if args.config == "c1":
        return (f"views-sharded x{world} (view v on rank v % {world}; one NCCL gather of the "
                f"views to rank 0)" if world > 1 else "8 views in one render launch")
    if args.config == "c4":
        return f"frames-sharded x{world} (both eyes of a frame on one GPU)"
    if args.shard == "peer" and world > 1:
        return (f"tiles-sharded x{world} (8x4 tiles t % {world}, stored into rank 0's maps by "
                f"the render kernels over NVLink)")
    if args.shard == "tiles" and world > 1:
        return f"tiles-sharded x{world} (8x4 tiles t % {world}, one NCCL gather per frame)"
    return f"frames-sharded x{world}"


def scaling(args, world) -> str:
    if args.config == "c1" or (args.shard in ("tiles", "peer") and world > 1):
        return "strong"
    return "weak"


def make_scene(args, world):
    from paper_2202_05628_b200 import synthetic as S

    n = max(args.steps + args.warmup, 1) * world
    if args.config == "c2":
        return S.make_scene("c3", frames=max(64, n))  # configs[3] sequence, configs[2] asset
    if args.config == "c0":
        return S.make_scene("c0", frames=n)
    if args.config == "c1":
        return S.make_scene("c1", frames=1)
    return S.make_scene("c4", frames=max(48, n))


def config_dict(sc, args, world) -> dict:
    """The workload description -- identical for both arms."""
    cams = sc.cameras[0]
    W, H = cams[0].width, cams[0].height
    views = len(cams) if args.config in ("c1", "c4") else 1
    return {"workload": WORKLOADS[args.config], "config": args.config, "image": [W, H],
            "views_per_step": views, "rays_per_view": W * H, "voxels": sc.n_voxels,
            "channels": sc.channels, "sh_degree": sc.degree, "joints": sc.rig.n_joints,
            "lambda_th": sc.lambda_th, "sigma_dep": sc.sigma_dep,
            "parallelism": parallelism(args, world),
            "l2": "flushed between timed steps (256 MB write); the FLUT exceeds L2"
            if args.config in ("c2", "c4") else "flushed between timed steps (256 MB write)"}


def rays_per_step(sc, args, world) -> int:
    """Rays the whole job renders per step."""
    cams = sc.cameras[0]
    per_view = cams[0].width * cams[0].height
    if args.config == "c1":
        return per_view * len(cams)
    if args.config == "c4":
        return per_view * len(cams) * world
    if args.shard in ("tiles", "peer") and world > 1:
        return per_view
    return per_view * world


# ---------------------------------------------------------------------------
# clocks, peaks, host description


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([c.strip() for c in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 5 + i and r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def physical_gpu(local: int) -> int:
    vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
    ids = [v for v in vis.split(",") if v.strip().isdigit()]
    return int(ids[local]) if local < len(ids) else local


def measured_peaks():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def ncu_traffic(config):
    p = os.path.join(REPO, "profiles", "render_traffic.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        if d.get("config", "c2") == config:
            return d
    return None


def host_cpu() -> dict:
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
    except Exception:
        pass
    return {"model": model, "logical_cpus": os.cpu_count(),
            "numpy": np.__version__}


# ---------------------------------------------------------------------------
# reference CPU path


def ref_frames(sc, args, frame_ids, nthreads=None):
    """Full frames of the step workload through the reference CPU path."""
    from paper_2202_05628_b200 import kinematics as KM
    import ref_port

    rf = ref_port.RefFrame(sc, nthreads=nthreads)
    per = []
    rays = 0
    for f in frame_ids:
        tables = KM.pose_tables(sc.rig, KM.PoseSpec.make(sc.poses[f]))
        cams = sc.cameras[f] if args.config in ("c1", "c4") else [sc.cameras[f][0]]
        t = rf.frame(tables, cams)
        per.append(t)
        rays = t["rays_sampled"]
    return rf, per, rays


def cpu_baseline(sc, args):
    n_all = len(sc.poses)
    frames = [f % n_all for f in range(max(1, args.cpu_frames))]
    if args.config == "c4":
        frames = frames[:1]
    rf, per, rays = ref_frames(sc, args, frames)
    tot = [t["warp"] + t["build-octree"] + t["volume-render"] for t in per]
    ms = statistics.median(tot) * 1e3
    out = {
        "value": rays / (ms / 1e3), "unit": "rays/s", "cores": rf.nthreads, "kind": rf.kind,
        "ms_per_step": ms,
        "stage_ms": {k: statistics.median(t[k] for t in per) * 1e3
                     for k in ("warp", "build-octree", "volume-render")},
        "host": host_cpu(),
        "sample": (f"{len(per)} full steps of the same workload ({rays} rays each, every "
                   f"pixel rendered, no extrapolation), median; reference kernels = "
                   f"{'oracle/_ref (reference _core.pyx, -O3 -fopenmp)' if rf.kind == 'reference' else 'oracle C port'}"
                   f" with {rf.nthreads} OpenMP threads, numpy stages from oracle/ref_port.py"),
    }
    if not args.no_cpu_1thread and args.config != "c4":
        rf1, per1, rays1 = ref_frames(sc, args, frames[:1], nthreads=1)
        t = per1[0]
        s1 = t["warp"] + t["build-octree"] + t["volume-render"]
        out["one_thread"] = {"value": rays1 / s1, "unit": "rays/s", "ms_per_step": s1 * 1e3,
                             "stage_ms": {k: t[k] * 1e3 for k in
                                          ("warp", "build-octree", "volume-render")},
                             "sample": "1 full step, ANIMVOX_THREADS=1 equivalent "
                                       "(nthreads=1 for every reference kernel)"}
    return out


def run_reference(args, world, rank):
    """--impl reference: the reference's CPU path on the host cores (rank 0)."""
    if rank != 0:
        return
    sc = make_scene(args, 1)
    n_all = len(sc.poses)
    warm = args.warmup if args.config != "c4" else min(args.warmup, 1)
    ids = [s % n_all for s in range(warm + args.steps)]
    rf, per, rays = ref_frames(sc, args, ids)
    per = per[warm:]
    steps = [t["warp"] + t["build-octree"] + t["volume-render"] for t in per]
    total = sum(steps)
    value = rays * len(steps) / total
    line = {
        "impl": "reference", "metric": METRICS[args.config], "value": value, "unit": "rays/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total / len(steps) * 1e3, "higher_is_better": True,
        "scaling": scaling(args, world), "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_dict(sc, args, world),
        "stage_ms": {k: statistics.median(t[k] for t in per) * 1e3
                     for k in ("warp", "build-octree", "volume-render")},
        "cpu_baseline": {"value": value, "unit": "rays/s", "cores": rf.nthreads,
                         "kind": rf.kind, "host": host_cpu(),
                         "sample": f"every step a full frame ({rays} rays, every pixel "
                                   f"rendered); warmup {warm} steps"},
        "e2e": {"value": value, "unit": "rays/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm


class Runner:
    """The step of each workload on this rank (graph-replayed, on fp.stream)."""

    def __init__(self, args, sc, fp, world, rank):
        import torch

        from paper_2202_05628_b200 import kinematics as KM

        self.args, self.sc, self.fp, self.world, self.rank = args, sc, fp, world, rank
        self.torch = torch
        self.KM = KM
        self.tiles = args.config in ("c0", "c2") and args.shard in ("tiles", "peer") and world > 1
        self.peer = self.tiles and args.shard == "peer"
        n = len(sc.poses)
        steps = args.warmup + args.steps
        if args.config == "c1":
            self.frames = [0] * steps
            self.my_views = [v for v in range(len(sc.cameras[0])) if v % world == rank]
        elif self.tiles:
            self.frames = [s % n for s in range(steps)]
        else:
            self.frames = [(rank + world * s) % n for s in range(steps)]
        self.tables = {f: KM.pose_tables(sc.rig, KM.PoseSpec.make(sc.poses[f]))
                       for f in set(self.frames)}
        self.poses = {f: KM.PoseSpec.make(sc.poses[f]) for f in set(self.frames)}
        self.cams = {f: [fp.camera(c) for c in sc.cameras[f]] for f in set(self.frames)}
        cam0 = sc.cameras[0][0]
        self.W, self.H = cam0.width, cam0.height
        if self.peer:
            from paper_2202_05628_b200 import parallel as PL
            self.asm = PL.PeerAssembly(fp, self.W, self.H)
        self.gather_buf = None

    def kw(self):
        return dict(lambda_th=self.sc.lambda_th, sigma_dep=self.sc.sigma_dep)

    def step(self, s, graph=True, outs=None):
        """Enqueue step s; returns the device tensors rank 0 reads back."""
        torch = self.torch
        fp = self.fp
        f = self.frames[s]
        pose, tables = self.poses[f], self.tables[f]
        if self.args.config == "c1":
            cams = [self.cams[f][v] for v in self.my_views]
            res = fp.run_views(pose, cams, graph=graph, tables=tables, outs=outs, **self.kw())
            return self.gather_views(res)
        if self.args.config == "c4":
            res = fp.run_views(pose, self.cams[f], graph=graph, tables=tables, outs=outs,
                               **self.kw())
            return [x for o in res for x in o]
        cam = self.cams[f][0]
        if self.peer:
            out = self.asm.frame(pose, cam, graph=graph, tables=tables, **self.kw())
            return list(out) if out is not None else []
        out = fp.run(pose, cam, graph=graph, tables=tables, out=outs[0] if outs else None,
                     tiles=(self.rank, self.world) if self.tiles else None, **self.kw())
        if self.tiles:
            from paper_2202_05628_b200 import parallel as PL
            with torch.cuda.stream(fp.stream):
                PL.assemble_tiles(*out, self.W, self.H, dst=0)
            return list(out) if self.rank == 0 else []
        return list(out)

    def gather_views(self, res):
        """configs[1]: ONE NCCL gather of every rank's views to rank 0."""
        torch = self.torch
        if self.world == 1:
            return [x for o in res for x in o]
        import torch.distributed as dist

        fp = self.fp
        n = self.W * self.H
        per_view = n * (self.sc.channels + 2)
        cap = -(-len(self.sc.cameras[0]) // self.world)
        with torch.cuda.stream(fp.stream):
            if self.gather_buf is None:
                self.gather_buf = torch.zeros(cap * per_view, dtype=torch.float32, device="cuda")
                self.gather_list = ([torch.empty_like(self.gather_buf)
                                     for _ in range(self.world)] if self.rank == 0 else None)
            for i, (F, A, D) in enumerate(res):
                b = self.gather_buf[i * per_view:(i + 1) * per_view]
                b[:n * self.sc.channels].copy_(F.reshape(-1))
                b[n * self.sc.channels:n * (self.sc.channels + 1)].copy_(A)
                b[n * (self.sc.channels + 1):].copy_(D)
            dist.gather(self.gather_buf, gather_list=self.gather_list, dst=0)
        return list(self.gather_list) if self.rank == 0 else []


def main():
    args = parse()
    maybe_spawn(args)
    world, rank, local = dist_env()
    if world != args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}\n")
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    import torch
    import torch.distributed as dist

    if torch.cuda.device_count() < 1:
        sys.stderr.write("bench.py: no CUDA device (the GPU arm has no CPU fallback)\n")
        sys.exit(2)
    # ARTEMIS_BENCH_SHARED_GPU=1: every rank on cuda:0 with gloo plumbing --
    # a launcher test on a one-GPU box for the collective-free shardings, never
    # a scaling measurement
    shared = os.environ.get("ARTEMIS_BENCH_SHARED_GPU") == "1"
    if shared and (args.config == "c1" or args.shard != "frames"):
        sys.stderr.write("bench.py: ARTEMIS_BENCH_SHARED_GPU only for frame sharding\n")
        sys.exit(2)
    if not shared and world > torch.cuda.device_count():
        sys.stderr.write(f"bench.py: {world} ranks but {torch.cuda.device_count()} GPUs\n")
        sys.exit(2)
    local = 0 if shared else local
    torch.cuda.set_device(local)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    red_dev = "cpu" if shared else "cuda"
    from paper_2202_05628_b200 import kernels as K
    from paper_2202_05628_b200 import kinematics as KM
    from paper_2202_05628_b200.frame import FramePipeline

    ranks = [{"rank": rank, "device": torch.cuda.get_device_name(local),
              "pci_bus": torch.cuda.get_device_properties(local).pci_bus_id
              if hasattr(torch.cuda.get_device_properties(local), "pci_bus_id") else None}]
    if world > 1:
        allr = [None] * world
        dist.all_gather_object(allr, ranks[0])
        ranks = allr

    sc = make_scene(args, world)
    fp = FramePipeline.from_scene(sc)
    run = Runner(args, sc, fp, world, rank)
    stream = fp.stream
    flush = torch.empty(FLUSH_BYTES, dtype=torch.uint8, device="cuda")
    rays_step = rays_per_step(sc, args, world)

    for s in range(args.warmup):  # under the timed conditions: L2 flushed before each step
        with torch.cuda.stream(stream):
            flush.fill_(s & 0xFF)
        run.step(s)
    stream.synchronize()
    launches = fp.launches_per_frame()

    # ---- timed region: K steps, device time via events, L2 flushed between
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    with ClockSampler(physical_gpu(local)) as clocks:
        for s in range(args.steps):
            with torch.cuda.stream(stream):
                flush.fill_(s & 0xFF)
            starts[s].record(stream)
            run.step(args.warmup + s)
            ends[s].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = [a.elapsed_time(b) for a, b in zip(starts, ends)]
    total_ms = sum(ms)
    t = torch.tensor([total_ms], dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    value = args.steps * rays_step / (total_ms / 1e3)

    # ---- stage breakdown (eager, profiled frames of view 0) -> roofline
    f0 = run.frames[0]
    cam0 = sc.cameras[f0][0]
    W, H = cam0.width, cam0.height
    fp.profile(True)
    stages = []
    for s in range(min(5, args.steps)):
        f = run.frames[s]
        with torch.cuda.stream(stream):
            flush.fill_(s & 0xFF)
        fp.run(run.poses[f], run.cams[f][0], graph=False, tables=run.tables[f], **run.kw())
        stages.append(fp.stage_ms())
    fp.profile(False)
    stage_ms = {k: statistics.mean(d[k] for d in stages) for k in stages[0]}
    n_in, n_live = fp.counts()
    # unique FLUT rows one view of frame 0 touches (diagnostic, untimed)
    fp.run(run.poses[f0], run.cams[f0][0], graph=False, parity=True, tables=run.tables[f0],
           **run.kw())
    tree = fp.tree()
    R, origin = cam0.cam_to_world()
    og, dg, dw = K.camera_rays_device(R, origin, cam0.fx, cam0.fy, cam0.cx, cam0.cy, W, H,
                                      sc.lo, sc.cell_size)
    shade = K.DeviceShading(np.zeros((sc.n_voxels, 2)), np.zeros(sc.n_voxels, np.int32),
                            np.eye(3)[None], 0, 1)
    dtree = K.DeviceTree(tree["codes"], tree["flut_idx"], tree["root"], tree["left"],
                         tree["right"], tree["box_min"], tree["box_size"], shade)
    rays_d = K.DeviceRays.from_tensors(og, dg, dw)
    counts = K.count_hits_device(dtree, rays_d)
    total_hits = int(counts.sum().item())
    hit_rays = int((counts > 0).sum().item())
    _, _, _, hidx, _, _ = K.forward_fit_device(dtree, shade, rays_d)
    unique_rows = int(torch.unique(hidx).numel())
    del og, dg, dw, dtree, shade, hidx, rays_d
    peak, peak_kind = measured_peaks()
    h = (sc.degree + 1) ** 2
    alg = unique_rows * (4 * h * sc.channels + 8 + 4) + 44 * n_live + W * H * 4 * (sc.channels + 2)
    achieved = alg / (stage_ms["render"] / 1e3) / 1e9
    traffic = ncu_traffic(args.config)

    e2e = e2e_api = None
    if not args.no_e2e:
        e2e = measure_e2e(args, sc, fp, run, world, rank, rays_step, red_dev)
        if args.config in ("c0", "c2") and world == 1:
            e2e_api = measure_e2e_api(args, sc, run)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(sc, args)
        except Exception as exc:  # the baseline must never sink the GPU line
            cpu = {"value": None, "unit": "rays/s", "cores": os.cpu_count(), "kind": "port",
                   "sample": f"failed: {exc!r}"}

    if rank == 0:
        line = {
            "metric": METRICS[args.config], "value": value, "unit": "rays/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": scaling(args, world),
            "vs_baseline": None, "dtype": "f64+f32", "data": "synthetic",
            "config": config_dict(sc, args, world),
            "stats": {"rays_per_step": rays_step, "live_leaves": n_live, "in_bounds": n_in,
                      "hit_rays_view0": hit_rays, "hits_view0": total_hits,
                      "unique_rows_view0": unique_rows, "graph": True},
            "ranks": ranks,
            "shared_gpu": shared,
            "stage_ms": stage_ms,
            "roofline": {"bound": "hbm", "kernel": "render_kernel", "achieved": achieved,
                         "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                         "frac": achieved / peak,
                         "traffic": traffic.get("bytes_per_launch") if traffic else None,
                         "alg_bytes": alg,
                         "per_unit": "U unique FLUT rows x (4*9*C + 12) B + 44 B x live "
                                     "leaves + 4(C+2) B x rays of one view (eager launch)"},
            "gpu_launches": launches * args.steps,
            "clocks": clocks.summary(),
            "e2e": e2e,
            "e2e_api": e2e_api,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    fp.close()
    if world > 1:
        dist.destroy_process_group()


def measure_e2e(args, sc, fp, run, world, rank, rays_step, red_dev="cuda"):
    """Steps through the public API with host buffers: host FK + pinned H2D of
    the pose/camera block + the device work (+ gather) + D2H of the result
    maps into pinned host memory; wall clock, max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_2202_05628_b200 import kinematics as KM

    K_ = args.steps
    frames = run.frames[args.warmup:args.warmup + K_]
    h2d = sc.rig.n_joints * 21 * 8 + C.sizeof(run.cams[frames[0]][0])
    if args.config in ("c0", "c2") and not run.tiles:
        # FramePipeline.run_stream: frame k renders while frame k-1 crosses PCIe
        items = [(KM.PoseSpec.make(sc.poses[f]), sc.cameras[f][0]) for f in frames]
        for _ in fp.run_stream(items[:2], **run.kw()):
            pass
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in fp.run_stream(items, **run.kw()):
            pass
        e2e_s = time.perf_counter() - t0
        d2h = int(statistics.mean(fp.last_stream_d2h_bytes))
        readout = ("dense F/alpha/depth maps in pinned host memory, refreshed by 2-D "
                   "copy-engine D2H of the union of this and the buffer's previous frame's "
                   "covered-pixel bounding box (bit-identical maps)")
    else:
        # tiles / views / stereo: host FK every step, the step (+ gather), then
        # every view's F/alpha/depth into persistent dense pinned host maps on
        # rank 0 (frame.ViewsReadout: per view the covered-pixel bounding box
        # united with the box that host buffer last received, as 2-D copies
        # on a copy stream -- outside the union both frames are (0, 0, +inf):
        # bit-identical dense maps). Pipelined: step k+1 renders while step
        # k's boxes cross PCIe (two device output sets, two host sets).
        cs = torch.cuda.Stream()
        Cc = sc.channels
        n = run.W * run.H
        outs = [None, None]
        if args.config in ("c1", "c4"):
            n_v = len(run.my_views) if args.config == "c1" else len(sc.cameras[0])
            outs = [fp.view_outputs(run.W, run.H, n_v),
                    [tuple(x.clone() for x in o) for o in fp.view_outputs(run.W, run.H, n_v)]]
        elif run.tiles and not run.peer:
            outs = [[fp.outputs(run.W, run.H)],
                    [tuple(x.clone() for x in fp.outputs(run.W, run.H))]]
        from paper_2202_05628_b200.frame import ViewsReadout

        readers = [None, None]
        # outputs shared by both sets: the root's peer maps, the gathered views
        shared_out = run.peer or (args.config == "c1" and world > 1)

        def triples_of(res):
            """Flat step results -> [(F (n, C), alpha (n), depth (n))] per view."""
            if args.config == "c1" and world > 1:
                per_view = n * (Cc + 2)
                out = []
                for r, buf in enumerate(res):
                    nv_r = len([v for v in range(len(sc.cameras[0])) if v % world == r])
                    for i in range(nv_r):
                        blk = buf[i * per_view:(i + 1) * per_view]
                        out.append((blk[:n * Cc].view(n, Cc), blk[n * Cc:n * (Cc + 1)],
                                    blk[n * (Cc + 1):]))
                return out
            return [tuple(res[3 * i:3 * i + 3]) for i in range(len(res) // 3)]

        def enqueue(s, b):
            for rd in (readers if shared_out else [readers[b]]):
                if rd is not None and rd.copied is not None:
                    fp.stream.wait_event(rd.copied)  # its previous D2H has read them
            f = run.frames[args.warmup + s]
            run.tables[f] = fp.tables(KM.PoseSpec.make(sc.poses[f]))  # host FK (canonical cached)
            tri = triples_of(run.step(args.warmup + s, outs=outs[b]))
            if not tri:
                return
            if readers[b] is None:
                readers[b] = ViewsReadout(tri, run.W, run.H, Cc)
            readers[b].mark(fp.stream)

        def finish(b):
            return readers[b].copy(cs) if readers[b] is not None else 0

        for w_ in range(2):  # warm both sets (graphs, pinned buffers)
            enqueue(w_, w_)
            finish(w_)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        moved = []
        t0 = time.perf_counter()
        for s in range(K_):
            enqueue(s, s % 2)
            if s > 0:
                moved.append(finish((s - 1) % 2))
        moved.append(finish((K_ - 1) % 2))
        torch.cuda.synchronize()
        e2e_s = time.perf_counter() - t0
        d2h = int(statistics.mean(moved)) if moved else 0
        readout = ("dense F/alpha/depth maps of every view in pinned host memory on rank 0, "
                   "refreshed by 2-D copy-engine D2H of the union of this and the buffer's "
                   "previous covered-pixel bounding box (bit-identical maps)")
    if world > 1:
        te = torch.tensor([e2e_s], dtype=torch.float64, device=red_dev)
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_s = float(te.item())
    return {"value": K_ * rays_step / e2e_s, "unit": "rays/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": e2e_s / K_ * 1e3, "readout": readout}


def measure_e2e_api(args, sc, run):
    """The reference's per-frame entry point as the installed CLI/service
    calls it (render.timed_render_frame -> pipeline.timed_render_frame):
    returns fp64 FrameBuffers in host memory; once per policy of the device
    asset cache (content digest of the asset arrays every call, or identity)."""
    from paper_2202_05628_b200 import kernels as K
    from paper_2202_05628_b200 import kinematics as KM
    from paper_2202_05628_b200 import pipeline as P
    from paper_2202_05628_b200 import types as T

    flut64 = sc.flut64()
    asset = T.CharacterAsset(
        voxels=T.VoxelSet(resolution=sc.resolution, bounds=T.Bounds(sc.lo, sc.hi),
                          cells=sc.cells),
        flut=T.FLUT(data=flut64, degree=sc.degree, channels=sc.channels),
        skeleton=sc.rig, weights=T.SkinWeights(joint_indices=sc.skin_idx, weights=sc.skin_w))
    opts = T.RenderOptions(lambda_th=sc.lambda_th, sigma_dep=sc.sigma_dep)
    frames = run.frames[args.warmup:args.warmup + args.steps]
    cam0 = sc.cameras[frames[0]][0]
    out = {}
    for policy in ("content", "identity"):
        K.set_cache_policy(policy)
        P.DEVICE_ASSETS.clear()
        for f in frames[:2]:  # warm: builds the resident pipeline and its graphs
            P.timed_render_frame(asset, KM.PoseSpec.make(sc.poses[f]), sc.cameras[f][0], opts)
        t0 = time.perf_counter()
        stages = []
        for f in frames:
            fb, st = P.timed_render_frame(asset, KM.PoseSpec.make(sc.poses[f]),
                                          sc.cameras[f][0], opts)
            stages.append(st)
        e = time.perf_counter() - t0
        out[policy] = {"value": len(frames) * cam0.width * cam0.height / e,
                       "ms_per_step": e / len(frames) * 1e3,
                       "stage_ms": {k: statistics.median(s[k] for s in stages) * 1e3
                                    for k in stages[0]}}
    K.set_cache_policy("content")
    P.DEVICE_ASSETS.clear()
    n = cam0.width * cam0.height
    return {"value": out["content"]["value"], "unit": "rays/s",
            "h2d_bytes_per_step": sc.rig.n_joints * 21 * 8 + 200,
            "d2h_bytes_per_step": n * (4 * sc.channels + 16),
            "ms_per_step": out["content"]["ms_per_step"],
            "call": "pipeline.timed_render_frame(asset, pose, camera, RenderOptions) -> "
                    "(FrameBuffers fp64 features/alpha/depth, stage seconds)",
            "content_policy": out["content"], "identity_policy": out["identity"],
            "note": "content policy: the asset arrays (fp64 FLUT included) are digested on "
                    "every call so in-place edits take effect, as in the reference"}


if __name__ == "__main__":
    main()
