"""Multi-GPU plumbing for the frame pipeline.

One process per GPU (torchrun), torch.distributed for the plumbing (NCCL
over NVLink on GPUs, gloo in CPU tests). Rays are independent, so the path
shards without any exchange inside a frame:

* frames  (configs[3], configs[4]): each rank warps, rebuilds and renders
          its own frames -- weak scaling, no data-path collective;
* views   (configs[1]): view v on rank v % world, same as frames;
* tiles   (configs[2]): every rank rebuilds the same posed tree and renders
          the 8x4-pixel tiles t with t % world == rank; each rank packs only
          those pixels into one contiguous shard (artemis_tiles_pack), ONE
          gather moves the shards to the root, and the root unpacks them
          into the image (artemis_tiles_unpack). Only rendered pixels cross
          NVLink ((world-1)/world of the frame), and the assembled frame is
          bit-identical to a single-GPU render;
          or, with PeerAssembly, no gather at all: every rank's render
          kernel writes its tiles' pixels straight into the root's
          full-frame buffers (CUDA IPC mapping, peer stores over NVLink),
          overlapping the transfer with the render ray by ray.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def world() -> tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def shard_frames(n_frames: int, rank: int, world_size: int) -> list[int]:
    """Round-robin frame (or view) ownership: frame f on rank f % world."""
    return [f for f in range(n_frames) if f % world_size == rank]


def frame_for_step(step: int, rank: int, world_size: int, n_frames: int) -> int:
    """Frame a rank renders at a given step of a weak-scaling run."""
    return (rank + world_size * step) % n_frames


def tile_owner(tile: int, world_size: int) -> int:
    return tile % world_size


def tile_shard(rank: int, world_size: int) -> tuple[int, int]:
    """(tile_start, tile_stride) for artemis_camera."""
    return (rank, world_size) if world_size > 1 else (0, 1)


def n_tiles(width: int, height: int) -> int:
    return ((width + 7) // 8) * ((height + 3) // 4)


def shard_floats(width: int, height: int, channels: int, start: int, stride: int) -> int:
    """Floats in one packed shard (artemis_tiles_shard_floats)."""
    t = n_tiles(width, height)
    return (max(0, (t - start + stride - 1) // stride) if start < t else 0) * 32 * (channels + 2)


def tile_pixels(width: int, height: int, start: int, stride: int) -> np.ndarray:
    """Host statement of the shard layout: pixel index (row-major) of every
    packed slot, -1 for slots outside the image. Slot s of the shard is
    pixel (s & 31) of tile start + (s >> 5) * stride, tile-row order."""
    tx = (width + 7) // 8
    t = np.arange(start, n_tiles(width, height), stride, dtype=np.int64)
    s = np.arange(32, dtype=np.int64)
    px = (t[:, None] % tx) * 8 + (s[None, :] & 7)
    py = (t[:, None] // tx) * 4 + (s[None, :] >> 3)
    pix = py * width + px
    return np.where((px < width) & (py < height), pix, -1).reshape(-1)


def gather_shards(packed: torch.Tensor, sizes: list[int], dst: int = 0):
    """ONE gather of every rank's packed shard to `dst` (shards padded to the
    largest size). Returns the list of per-rank shards on dst, None elsewhere."""
    rank, ws = world()
    cap = max(sizes)
    if packed.numel() < cap:
        buf = torch.zeros(cap, dtype=packed.dtype, device=packed.device)
        buf[:packed.numel()] = packed
    else:
        buf = packed
    gl = [torch.empty_like(buf) for _ in range(ws)] if rank == dst else None
    dist.gather(buf, gather_list=gl, dst=dst)
    if rank != dst:
        return None
    return [g[:sizes[r]] for r, g in enumerate(gl)]


def assemble_tiles(F: torch.Tensor, alpha: torch.Tensor, depth: torch.Tensor, width: int,
                   height: int, dst: int = 0):
    """Assemble a tile-sharded frame on `dst` in place: every rank's F/alpha/
    depth holds its own tiles (render with tiles=tile_shard(rank, world));
    on return dst's buffers hold the whole image. Device tensors (CUDA)."""
    from . import _lib
    from ._lib import check
    from .device import ptr

    rank, ws = world()
    if ws == 1:
        return F, alpha, depth
    L = _lib.lib()
    C = F.numel() // (width * height)
    st = torch.cuda.current_stream().cuda_stream or None
    sizes = [shard_floats(width, height, C, r, ws) for r in range(ws)]
    packed = torch.empty(max(sizes[rank], 1), dtype=torch.float32, device=F.device)
    if sizes[rank]:
        check(L.artemis_tiles_pack(ptr(F), ptr(alpha), ptr(depth), width, height, C, rank, ws,
                                   ptr(packed), st), "tiles_pack")
    shards = gather_shards(packed[:sizes[rank]], sizes, dst)
    if rank == dst:
        for r, sh in enumerate(shards):
            if r == dst or not sizes[r]:
                continue
            check(L.artemis_tiles_unpack(ptr(sh), width, height, C, r, ws, ptr(F), ptr(alpha),
                                         ptr(depth), st), "tiles_unpack")
    return F, alpha, depth


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (device timings are reported as the max)."""
    rank, ws = world()
    if ws == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _camera_size(camera) -> tuple[int, int]:
    return int(camera.width), int(camera.height)


class PeerAssembly:
    """Tile-sharded frames assembled by the render kernels themselves.

    The root (`dst`) owns full-frame F / alpha / depth device tensors; every
    other rank maps them into its address space (CUDA IPC handles, exchanged
    once through torch.distributed) and hands them to its FramePipeline
    (artemis_frame_set_output_peer). A frame is then: root initialises the
    maps -> barrier -> every rank renders its tiles (t % world == rank),
    its kernel storing each finished ray's pixels directly into the root's
    maps over NVLink -> stream sync + barrier -> the root holds the whole
    image. No pack, no collective on the data path, no unpack; bit-identical
    to a single-GPU render (every pixel is written by exactly one rank)."""

    def __init__(self, fp, width: int, height: int, *, maps64: bool = False, dst: int = 0):
        from torch.multiprocessing.reductions import reduce_tensor

        self.fp, self.width, self.height, self.dst = fp, int(width), int(height), dst
        self.rank, self.world = world()
        n = self.width * self.height
        mt = torch.float64 if maps64 else torch.float32
        self.maps64 = maps64
        if self.rank == dst:
            self.F = torch.zeros((n, fp.channels), dtype=torch.float32, device="cuda")
            self.A = torch.zeros(n, dtype=mt, device="cuda")
            self.D = torch.full((n,), float("inf"), dtype=mt, device="cuda")
            shared = [[reduce_tensor(t) for t in (self.F, self.A, self.D)]]
        else:
            shared = [None]
        if self.world > 1:
            dist.broadcast_object_list(shared, src=dst)
        if self.rank != dst:
            self.F, self.A, self.D = (fn(*args) for fn, args in shared[0])
        fp.set_output_peer(self.F, self.A, self.D)

    def frame(self, pose, camera, **kw):
        """Render one tile-sharded frame into the root's maps; returns the
        root's (F, alpha, depth) on the root, None elsewhere. With one rank
        the frame is rendered unsharded into the pipeline's own maps."""
        w, h = _camera_size(camera)
        if (w, h) != (self.width, self.height):
            raise ValueError(f"camera is {w}x{h}; the assembly maps are "
                             f"{self.width}x{self.height}")
        if self.world == 1:
            F, A, D = self.fp.run(pose, camera, maps64=self.maps64, **kw)
            self.fp.stream.synchronize()
            return F, A, D
        if self.rank == self.dst:
            with torch.cuda.stream(self.fp.stream):
                self.F.zero_()
                self.A.zero_()
                self.D.fill_(float("inf"))
        self.fp.stream.synchronize()
        if self.world > 1:
            dist.barrier()  # the root's maps are initialised before any rank stores
        self.fp.run(pose, camera, tiles=tile_shard(self.rank, self.world), maps64=self.maps64,
                    **kw)
        self.fp.stream.synchronize()
        if self.world > 1:
            dist.barrier()  # every rank's stores have landed
        return (self.F, self.A, self.D) if self.rank == self.dst else None

    def close(self):
        """Detach the pipeline from the peer maps. Every rank drops its IPC
        mapping before the root may free the maps (barrier), so no process
        tears down memory another one still maps."""
        self.fp.set_output_peer(None)
        self.fp.stream.synchronize()
        if self.rank != self.dst:
            self.F = self.A = self.D = None
            torch.cuda.synchronize()
        if self.world > 1:
            dist.barrier()
