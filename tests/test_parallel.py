"""Multi-process (gloo, world_size 2) checks of the N>1 host logic: frame
sharding, max-over-ranks timing and the exact tile-assembly reduction."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2202_05628_b200 import parallel as PL


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def tile_mask(width, height, rank, world):
    """Pixels of the 8x4 tiles owned by `rank` (tile t on rank t % world)."""
    tx = (width + 7) // 8
    ys, xs = np.mgrid[0:height, 0:width]
    tile = (ys // 4) * tx + xs // 8
    return (tile % world == rank).reshape(-1)


def _worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        W, H, C = 37, 21, 5
        rng = np.random.default_rng(7)
        F = rng.normal(size=(W * H, C)).astype(np.float32)
        A = rng.uniform(size=W * H).astype(np.float32)
        D = np.where(rng.uniform(size=W * H) < 0.3, rng.uniform(1, 3, W * H), np.inf)
        D = D.astype(np.float32)
        own = tile_mask(W, H, rank, world)
        Fp = torch.from_numpy(np.where(own[:, None], F, 0.0).astype(np.float32))
        Ap = torch.from_numpy(np.where(own, A, 0.0).astype(np.float32))
        Dp = torch.from_numpy(np.where(own, D, np.inf).astype(np.float32))
        PL.assemble_tiles(Fp, Ap, Dp, dst=0)
        t = PL.max_over_ranks(float(rank + 1))
        frames = PL.shard_frames(10, rank, world)
        if rank == 0:
            out_q.put(("ok", np.array_equal(Fp.numpy(), F), np.array_equal(Ap.numpy(), A),
                       np.array_equal(Dp.numpy(), D), t))
        out_q.put(("frames", rank, frames))
    finally:
        dist.destroy_process_group()


def test_two_rank_assembly_and_sharding():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    msgs = [q.get(timeout=5) for _ in range(3)]
    ok = [m for m in msgs if m[0] == "ok"][0]
    assert ok[1] and ok[2] and ok[3], "tile assembly must reproduce the full frame exactly"
    assert ok[4] == 2.0
    frames = sorted(f for m in msgs if m[0] == "frames" for f in m[2])
    assert frames == list(range(10))


def test_single_process_helpers():
    assert PL.tile_shard(0, 1) == (0, 1)
    assert PL.tile_shard(3, 8) == (3, 8)
    assert [PL.frame_for_step(s, 1, 4, 64) for s in range(3)] == [1, 5, 9]
    assert PL.shard_frames(5, 0, 1) == [0, 1, 2, 3, 4]
    masks = [tile_mask(64, 32, r, 3) for r in range(3)]
    assert np.array_equal(sum(m.astype(int) for m in masks), np.ones(64 * 32, int))
