"""Multi-process (gloo, world_size 2) checks of the N>1 host logic: frame
sharding, max-over-ranks timing and the tile-shard gather (the packed shard
layout is stated on the host by parallel.tile_pixels; the CUDA pack/unpack
kernels are checked against it in test_gpu_pipeline.py)."""

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
        # each rank packs the pixels of its own tiles (host statement of the
        # artemis_tiles_pack layout), one gather, the root unpacks
        P = np.concatenate([F, A[:, None], D[:, None]], axis=1)
        sizes = [PL.shard_floats(W, H, C, r, world) for r in range(world)]
        pix = PL.tile_pixels(W, H, rank, world)
        mine = np.where(pix[:, None] >= 0, P[np.maximum(pix, 0)], 0.0).astype(np.float32)
        assert mine.size == sizes[rank]
        shards = PL.gather_shards(torch.from_numpy(mine.reshape(-1)), sizes, dst=0)
        if rank == 0:
            out = np.zeros_like(P)
            for r, sh in enumerate(shards):
                pr = PL.tile_pixels(W, H, r, world)
                v = sh.numpy().reshape(-1, C + 2)
                out[pr[pr >= 0]] = v[pr >= 0]
            Fp, Ap, Dp = (torch.from_numpy(np.ascontiguousarray(out[:, :C])),
                          torch.from_numpy(np.ascontiguousarray(out[:, C])),
                          torch.from_numpy(np.ascontiguousarray(out[:, C + 1])))
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
    assert ok[1] and ok[2] and ok[3], "tile gather must reproduce the full frame exactly"
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


def test_shard_layout_partitions_the_image():
    for W, H, ws in [(37, 21, 2), (64, 32, 3), (1024, 1024, 8), (5, 3, 4)]:
        seen = np.zeros(W * H, int)
        for r in range(ws):
            pix = PL.tile_pixels(W, H, r, ws)
            assert pix.size * (7 + 2) == PL.shard_floats(W, H, 7, r, ws)
            own = pix[pix >= 0]
            assert np.array_equal(np.sort(own), np.flatnonzero(tile_mask(W, H, r, ws)))
            seen[own] += 1
        assert (seen == 1).all()
