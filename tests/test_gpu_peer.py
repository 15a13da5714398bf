"""Tile-sharded frames assembled by peer stores (parallel.PeerAssembly):
two processes share the one GPU of the test box (no kernel waits on
another: the barriers are host-side gloo), rank 1 maps rank 0's full-frame
maps over CUDA IPC and its render kernel writes its tiles into them. The
assembled frame must equal a single-process render bit for bit."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_path, maps64):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2202_05628_b200 import kinematics as KM
    from paper_2202_05628_b200 import parallel as PL
    from paper_2202_05628_b200 import synthetic as S
    from paper_2202_05628_b200.frame import FramePipeline

    sc = S.make_scene("c0", resolution=64, image=(61, 45), frames=2)
    fp = FramePipeline.from_scene(sc)
    asm = PL.PeerAssembly(fp, 61, 45, maps64=maps64)
    outs = []
    for f in range(2):
        got = asm.frame(KM.PoseSpec.make(sc.poses[f]), sc.cameras[f][0], graph=f == 1)
        if rank == 0:
            outs.append([t.cpu().numpy().copy() for t in got])
    if rank == 0:
        ref = FramePipeline.from_scene(sc)
        for f in range(2):
            want = ref.run(KM.PoseSpec.make(sc.poses[f]), sc.cameras[f][0], graph=False,
                           maps64=maps64)
            ref.stream.synchronize()
            for a, b in zip(outs[f], want):
                assert np.array_equal(a, b.cpu().numpy()), f
        ref.close()
        open(out_path, "w").write("ok")
    dist.barrier()
    asm.close()  # mappings released on every rank before the root's maps go
    fp.close()
    del asm
    torch.cuda.synchronize()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("maps64", [False, True])
def test_peer_assembly_equals_single_render(tmp_path, maps64):
    out = tmp_path / "result"
    mp.spawn(_worker, args=(2, _port(), str(out), maps64), nprocs=2, join=True)
    assert out.read_text() == "ok"
