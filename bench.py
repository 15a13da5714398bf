"""Benchmark: full posed frames (LBS warp + Morton-key octree rebuild +
render) of the ~1M-leaf configs[2] character at 1024x1024, one frame per
step, poses/cameras from the configs[3] animation sequence on that asset.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl artemis|reference]

One process per GPU (torchrun for N > 1, NCCL); each rank renders its own
frames of the sequence (frames sharded, no data-path collective: weak
scaling). Rank 0 prints ONE JSON line. See DESIGN.md "Measurement".

  value       rays/s over all ranks = N * K * W*H / max-over-ranks device
              time of the K timed frames (CUDA events on the pipeline's
              stream; inputs resident in HBM; L2 flushed between frames)
  e2e         the same metric through the public Python API with host
              buffers: per frame, host FK -> H2D of the pose/camera block ->
              frame -> D2H of F/alpha/depth into pinned memory
  roofline    render kernel (the dominant kernel): algorithmic bytes per
              launch (U unique FLUT rows touched x (4*H*C + 12) + 44 B x
              live leaves + 4(C+2) B x rays) / its mean CUDA-event duration
  cpu_baseline  the reference's CPU path (its compiled kernels from
              oracle/_ref, numpy stages restated in oracle/ref_port.py) on a
              bounded sample, rank 0 at N = 1 only
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))

METRIC = "rays/s (full warp+rebuild+render frame, ~1M-leaf octree, 1024x1024)"
WORKLOAD = ("configs[2] asset (512^3 grid, 4-voxel shell, ~985k canonical voxels, 32-channel SH "
            "deg 2, 24 joints) rendered 1024x1024, one full posed frame per step with the "
            "configs[3] pose/camera sequence")
FLUSH_BYTES = 256 << 20  # > 126 MB L2


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="artemis", choices=["artemis", "reference"])
    ap.add_argument("--config", default="c2", choices=["c0", "c2"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-frames", type=int, default=2)
    ap.add_argument("--shard", default="frames", choices=["frames", "tiles", "peer"],
                    help="N>1: frames (weak scaling, no collective), 8x4 screen tiles of "
                         "the same frame (strong scaling, one NCCL gather per frame), or "
                         "tiles stored by the render kernels straight into rank 0's maps "
                         "over NVLink (peer: CUDA IPC mapping, no gather)")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def make_scene(name, frames):
    from paper_2202_05628_b200 import synthetic as S

    if name == "c2":
        return S.make_scene("c3", frames=frames)  # configs[3] sequence on the configs[2] asset
    return S.make_scene("c0", frames=frames)


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


def render_bytes(sc, n_live, unique_rows, rays):
    h = (sc.degree + 1) ** 2
    return unique_rows * (4 * h * sc.channels + 8 + 4) + 44 * n_live + rays * 4 * (sc.channels + 2)


def measured_peaks():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def ncu_traffic():
    p = os.path.join(REPO, "profiles", "render_traffic.json")
    if os.path.exists(p):
        with open(p) as fh:
            return json.load(fh)
    return None


def cpu_baseline(sc, frames, n_frames):
    from paper_2202_05628_b200 import kinematics as KM
    import ref_port

    rf = ref_port.RefFrame(sc)
    stride = 8
    times = []
    for f in range(n_frames):
        tables = KM.pose_tables(sc.rig, KM.PoseSpec.make(sc.poses[f]))
        t = rf.frame(tables, sc.cameras[f][0], row_stride=stride)
        times.append(t)
    cam = sc.cameras[0][0]
    rays = cam.width * cam.height
    per = [t["warp"] + t["build-octree"] + t["volume-render"] for t in times]
    ms = statistics.median(per) * 1e3
    return {
        "value": rays / (ms / 1e3), "unit": "rays/s", "cores": rf.nthreads, "kind": rf.kind,
        "ms_per_frame": ms,
        "stage_ms": {k: statistics.median(t[k] for t in times) * 1e3
                     for k in ("warp", "build-octree", "volume-render")},
        "sample": (f"{n_frames} full frames of the same workload; warp + resolve + build on all "
                   f"voxels, render on every {stride}th image row ({times[0]['rays_sampled']} "
                   f"rays) scaled to {rays} rays; reference kernels = "
                   f"{'oracle/_ref (reference _core.pyx, -O3 -fopenmp)' if rf.kind == 'reference' else 'oracle C port'}"
                   f", numpy stages from oracle/ref_port.py"),
    }


def run_reference(args, world, rank):
    """--impl reference: the reference's CPU path on the host cores."""
    if rank != 0:
        return
    sc = make_scene(args.config, max(1, args.steps + args.warmup))
    from paper_2202_05628_b200 import kinematics as KM
    import ref_port

    rf = ref_port.RefFrame(sc)
    stride = 8
    per = []
    for s in range(args.warmup + args.steps):
        f = s % len(sc.poses)
        tables = KM.pose_tables(sc.rig, KM.PoseSpec.make(sc.poses[f]))
        t = rf.frame(tables, sc.cameras[f][0], row_stride=stride)
        if s >= args.warmup:
            per.append(t["warp"] + t["build-octree"] + t["volume-render"])
    cam = sc.cameras[0][0]
    rays = cam.width * cam.height
    total = sum(per)
    value = rays * len(per) / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "rays/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total / len(per) * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "rays_per_frame": rays, "voxels": sc.n_voxels},
        "cpu_baseline": {"value": value, "unit": "rays/s", "cores": rf.nthreads, "kind": rf.kind,
                         "sample": f"every {stride}th image row rendered per frame, scaled to "
                                   f"{rays} rays; warp/resolve/build on all voxels"},
        "e2e": {"value": value, "unit": "rays/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    world, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    import torch
    import torch.distributed as dist

    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    from paper_2202_05628_b200 import kinematics as KM
    from paper_2202_05628_b200.frame import FramePipeline

    n_frames = args.warmup + args.steps
    sc = make_scene(args.config, max(64, n_frames * world) if args.config == "c2" else n_frames)
    frames = [(rank + world * s) % len(sc.poses) for s in range(n_frames)]
    tiles = args.shard in ("tiles", "peer") and world > 1
    peer = args.shard == "peer" and world > 1
    if tiles:  # every rank renders the same frame sequence, its own tiles
        frames = [s % len(sc.poses) for s in range(n_frames)]
        from paper_2202_05628_b200 import parallel as PL
    tables = {f: KM.pose_tables(sc.rig, KM.PoseSpec.make(sc.poses[f])) for f in set(frames)}
    fp = FramePipeline.from_scene(sc)
    cams = {f: fp.camera(sc.cameras[f][0]) for f in set(frames)}
    W, H = sc.cameras[0][0].width, sc.cameras[0][0].height
    rays = W * H
    stream = fp.stream
    flush = torch.empty(FLUSH_BYTES, dtype=torch.uint8, device="cuda")
    asm = PL.PeerAssembly(fp, W, H) if peer else None

    def frame(f, graph=True):
        if peer:
            return asm.frame(KM.PoseSpec.make(sc.poses[f]), cams[f], lambda_th=sc.lambda_th,
                             sigma_dep=sc.sigma_dep, graph=graph, tables=tables[f])
        out = fp.run(KM.PoseSpec.make(sc.poses[f]), cams[f],
                     lambda_th=sc.lambda_th, sigma_dep=sc.sigma_dep, graph=graph,
                     tables=tables[f], tiles=(rank, world) if tiles else None)
        if tiles:
            with torch.cuda.stream(stream):
                PL.assemble_tiles(*out, W, H, dst=0)
        return out

    for s in range(args.warmup):  # under the timed conditions: L2 flushed before each frame
        with torch.cuda.stream(stream):
            flush.fill_(s & 0xFF)
        frame(frames[s])
    stream.synchronize()
    launches = fp.launches_per_frame()

    # ---- timed region: K frames, device time via events, L2 flushed between
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
            frame(frames[args.warmup + s])
            ends[s].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = [a.elapsed_time(b) for a, b in zip(starts, ends)]
    total_ms = sum(ms)
    t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    value = (1 if tiles else world) * args.steps * rays / (total_ms / 1e3)

    # ---- stage breakdown (eager, profiled) -> roofline of the render kernel
    fp.profile(True)
    stages = []
    for s in range(min(5, args.steps)):
        with torch.cuda.stream(stream):
            flush.fill_(s & 0xFF)
        fp.run(KM.PoseSpec.make(sc.poses[frames[s]]), cams[frames[s]], lambda_th=sc.lambda_th,
               sigma_dep=sc.sigma_dep, graph=False, tables=tables[frames[s]])
        stages.append(fp.stage_ms())
    fp.profile(False)
    stage_ms = {k: statistics.mean(d[k] for d in stages) for k in stages[0]}
    n_in, n_live = fp.counts()

    # unique FLUT rows touched by one frame (diagnostic pass, untimed)
    from paper_2202_05628_b200 import kernels as K
    fp.run(KM.PoseSpec.make(sc.poses[frames[0]]), cams[frames[0]], graph=False, parity=True,
           tables=tables[frames[0]], lambda_th=sc.lambda_th, sigma_dep=sc.sigma_dep)
    tree = fp.tree()
    cam0 = sc.cameras[frames[0]][0]
    R, origin = cam0.cam_to_world()
    og, dg, dw = K.camera_rays_device(R, origin, cam0.fx, cam0.fy, cam0.cx, cam0.cy, W, H,
                                      sc.lo, sc.cell_size)
    shade = K.DeviceShading(np.zeros((sc.n_voxels, 2)), np.zeros(sc.n_voxels, np.int32),
                            np.eye(3)[None], 0, 1)
    dtree = K.DeviceTree(tree["codes"], tree["flut_idx"], tree["root"], tree["left"],
                         tree["right"], tree["box_min"], tree["box_size"], shade)
    counts = K.count_hits_device(dtree, K.DeviceRays.from_tensors(og, dg, dw))
    total_hits = int(counts.sum().item())
    hit_rays = int((counts > 0).sum().item())
    # rows touched: leaves with at least one hit (trace of the frame)
    _, _, _, hidx, _, _ = K.forward_fit_device(dtree, shade, K.DeviceRays.from_tensors(og, dg, dw))
    unique_rows = int(torch.unique(hidx).numel())
    del og, dg, dw, dtree, shade, hidx
    peak, peak_kind = measured_peaks()
    alg = render_bytes(sc, n_live, unique_rows, rays)
    achieved = alg / (stage_ms["render"] / 1e3) / 1e9
    traffic = ncu_traffic()

    # ---- e2e through the public API with host buffers
    e2e = None
    if not args.no_e2e and not tiles:
        h2d = sc.rig.n_joints * 21 * 8 + C.sizeof(cams[frames[0]])
        e2e_steps = args.steps
        items = [(KM.PoseSpec.make(sc.poses[f]), sc.cameras[f][0])
                 for f in frames[args.warmup:args.warmup + e2e_steps]]
        for _ in fp.run_stream(items[:2], lambda_th=sc.lambda_th, sigma_dep=sc.sigma_dep):
            pass  # warm the double-buffered graphs
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        # public API: host FK + pinned H2D of pose/camera + frame + D2H of
        # F/alpha/depth into pinned host memory, every frame
        for hF, hA, hD in fp.run_stream(items, lambda_th=sc.lambda_th, sigma_dep=sc.sigma_dep):
            pass
        e2e_s = time.perf_counter() - t0
        if world > 1:  # the job's end-to-end time is its slowest rank's
            te = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
            e2e_s = float(te.item())
        d2h = int(statistics.mean(fp.last_stream_d2h_bytes))
        e2e = {"value": world * e2e_steps * rays / e2e_s, "unit": "rays/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": e2e_s / e2e_steps * 1e3,
               "readout": "dense F/alpha/depth maps in pinned host memory, refreshed by 2-D "
                          "copy-engine D2H of the union of this and the buffer's previous "
                          "frame's covered-pixel bounding box (bit-identical maps)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(sc, frames, args.cpu_frames)
        except Exception as exc:  # the baseline must never sink the GPU line
            cpu = {"value": None, "unit": "rays/s", "cores": os.cpu_count(), "kind": "port",
                   "sample": f"failed: {exc!r}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "rays/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "strong" if tiles else "weak",
            "vs_baseline": None, "dtype": "f64+f32",
            "data": "synthetic",
            "config": {"workload": WORKLOAD, "image": [W, H], "rays_per_frame": rays,
                       "voxels": sc.n_voxels, "live_leaves": n_live, "in_bounds": n_in,
                       "channels": sc.channels, "sh_degree": sc.degree,
                       "frames_per_rank": args.steps,
                       "parallelism": (f"tiles-sharded x{world} (8x4 tiles t % {world}, "
                                       f"stored into rank 0's maps by the render kernels over "
                                       f"NVLink)" if peer else
                                       f"tiles-sharded x{world} (8x4 tiles t % {world}, one "
                                       f"NCCL gather per frame)" if tiles
                                       else f"frames-sharded x{world}"),
                       "l2": "flushed between timed frames (256 MB write)",
                       "graph": True, "hit_rays": hit_rays, "hits": total_hits,
                       "unique_rows": unique_rows},
            "stage_ms": stage_ms,
            "roofline": {"bound": "hbm", "kernel": "render_kernel", "achieved": achieved,
                         "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                         "frac": achieved / peak,
                         "traffic": traffic.get("bytes_per_launch") if traffic else None,
                         "alg_bytes": alg},
            "gpu_launches": launches * args.steps,
            "clocks": clocks.summary(),
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    fp.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
