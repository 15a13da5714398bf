"""Tile-order probe (configs[2]/[3] sequence): does starting the tiles with
the longest rays first shorten the render's tail? Per-pixel hit counts of
frame 0 (count_hits_device) -> per 8x4 tile max / sum -> candidate orders
installed with FramePipeline.set_tile_order; graph-replayed frames, L2
flushed between frames, CUDA events. The order never changes the maps."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2202_05628_b200 import kernels as K  # noqa: E402
from paper_2202_05628_b200 import kinematics as KM  # noqa: E402
from paper_2202_05628_b200 import synthetic as S  # noqa: E402
from paper_2202_05628_b200.frame import FramePipeline  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
NF = 20
sc = S.make_scene(name, frames=NF)
fp = FramePipeline.from_scene(sc)
poses = [KM.PoseSpec.make(sc.poses[f]) for f in range(NF)]
tabs = [fp.tables(p) for p in poses]
cams = [sc.cameras[f][0] for f in range(NF)]
W, H = cams[0].width, cams[0].height
tx, ty = (W + 7) // 8, (H + 3) // 4


def tile_hits(f):
    fp.run(poses[f], cams[f], graph=False, parity=True, tables=tabs[f])
    torch.cuda.synchronize()
    tree = fp.tree()
    shade = K.DeviceShading(np.zeros((sc.n_voxels, 2)), np.zeros(sc.n_voxels, np.int32),
                            np.eye(3)[None], 0, 1)
    dtree = K.DeviceTree(tree["codes"], tree["flut_idx"], tree["root"], tree["left"],
                         tree["right"], tree["box_min"], tree["box_size"], shade)
    R, origin = cams[f].cam_to_world()
    og, dg, dw = K.camera_rays_device(R, origin, cams[f].fx, cams[f].fy, cams[f].cx, cams[f].cy,
                                      W, H, sc.lo, sc.cell_size)
    counts = K.count_hits_device(dtree, K.DeviceRays.from_tensors(og, dg, dw))
    c = np.asarray(counts.cpu() if hasattr(counts, "cpu") else counts).reshape(H, W)
    cp = np.zeros((ty * 4, tx * 8), c.dtype)
    cp[:H, :W] = c
    t = cp.reshape(ty, 4, tx, 8).transpose(0, 2, 1, 3).reshape(ty * tx, 32)
    return t.max(1), t.sum(1)


mx, sm = tile_hits(0)
ids = np.arange(tx * ty)
cy_, cx_ = (ids // tx) * 4 + 2 - H / 2, (ids % tx) * 8 + 4 - W / 2
centre = np.lexsort((ids, np.hypot(cx_, cy_))).astype(np.int32)
orders = {
    "rowmajor": ids.astype(np.int32),
    "centre": centre,
    "maxdesc": np.lexsort((np.hypot(cx_, cy_), -mx)).astype(np.int32),
    "sumdesc": np.lexsort((np.hypot(cx_, cy_), -sm)).astype(np.int32),
    # long rays first, then the rest centre-out
    "max>=64first": np.concatenate([np.lexsort((np.hypot(cx_, cy_), -mx))[:int((mx >= 64).sum())],
                                    centre[np.isin(centre, np.where(mx < 64)[0])]]).astype(np.int32),
}
print(f"tiles {tx * ty}, max hits per ray {mx.max()}, tiles with a ray >= 64 hits {(mx >= 64).sum()}, "
      f">= 128 {(mx >= 128).sum()}", flush=True)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for rep in range(2):
    for oname, o in orders.items():
        fp.set_tile_order(W, H, o)
        for f in range(3):
            fp.run(poses[f], cams[f], tables=tabs[f])
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(NF)]
        for f in range(NF):
            with torch.cuda.stream(fp.stream):
                flush.fill_(f & 0xFF)
            ev[f][0].record(fp.stream)
            fp.run(poses[f], cams[f], tables=tabs[f])
            ev[f][1].record(fp.stream)
        torch.cuda.synchronize()
        ms = [a.elapsed_time(b) for a, b in ev]
        print(f"{oname:14s} {np.mean(ms):.4f} ms/frame (first 5 {np.mean(ms[:5]):.4f})", flush=True)
