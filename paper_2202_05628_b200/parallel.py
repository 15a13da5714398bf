"""Multi-GPU plumbing for the frame pipeline.

One process per GPU (torchrun), torch.distributed for the plumbing (NCCL
over NVLink on GPUs, gloo in CPU tests). Rays are independent, so the path
shards without any exchange inside a frame:

* frames  (configs[3], configs[4]): each rank warps, rebuilds and renders
          its own frames -- weak scaling, no data-path collective;
* tiles   (configs[2]): every rank rebuilds the same posed tree and renders
          the 8x4-pixel tiles t with t % world == rank; one reduction then
          assembles the image on the root: F and alpha are SUM-reduced
          (other ranks' pixels are exactly 0) and depth MIN-reduced (other
          ranks' pixels are +inf), so the assembled frame is bit-identical
          to a single-GPU render.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def world() -> tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def shard_frames(n_frames: int, rank: int, world_size: int) -> list[int]:
    """Round-robin frame ownership (frame f on rank f % world)."""
    return [f for f in range(n_frames) if f % world_size == rank]


def frame_for_step(step: int, rank: int, world_size: int, n_frames: int) -> int:
    """Frame a rank renders at a given step of a weak-scaling run."""
    return (rank + world_size * step) % n_frames


def tile_owner(tile: int, world_size: int) -> int:
    return tile % world_size


def tile_shard(rank: int, world_size: int) -> tuple[int, int]:
    """(tile_start, tile_stride) for artemis_camera."""
    return (rank, world_size) if world_size > 1 else (0, 1)


def assemble_tiles(F: torch.Tensor, alpha: torch.Tensor, depth: torch.Tensor, dst: int = 0):
    """Combine tile-sharded partial frames onto `dst` in place (one
    reduction per buffer; exact because the shards are disjoint)."""
    rank, ws = world()
    if ws == 1:
        return F, alpha, depth
    dist.reduce(F, dst=dst, op=dist.ReduceOp.SUM)
    dist.reduce(alpha, dst=dst, op=dist.ReduceOp.SUM)
    dist.reduce(depth, dst=dst, op=dist.ReduceOp.MIN)
    return F, alpha, depth


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (device timings are reported as the max)."""
    rank, ws = world()
    if ws == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
