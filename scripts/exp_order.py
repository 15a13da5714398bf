"""Timing experiment (variants/libartemis_order.so): render time with the
8x4 tiles visited in other orders -- most expensive first (from a previous
render's per-tile hit counts), centre-out, and the default row-major."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2202_05628_b200 import _lib  # noqa: E402
from paper_2202_05628_b200 import kinematics as KM  # noqa: E402
from paper_2202_05628_b200 import synthetic as S  # noqa: E402
from paper_2202_05628_b200.frame import FramePipeline  # noqa: E402

sc = S.make_scene("c3", frames=2)
fp = FramePipeline.from_scene(sc)
pose, cam = KM.PoseSpec.make(sc.poses[0]), sc.cameras[0][0]
W, H = cam.width, cam.height
fn = _lib.lib().artemis_debug_tile_order
fn.argtypes = [C.c_void_p]
fp.profile(True)


def render():
    ts = []
    for _ in range(7):
        fp.run(pose, cam, lambda_th=sc.lambda_th, sigma_dep=sc.sigma_dep, graph=False)
        ts.append(fp.stage_ms()["render"])
    return sorted(ts)[3]


fn(None)
F, A, D = [x.clone() for x in fp.run(pose, cam, lambda_th=sc.lambda_th, sigma_dep=sc.sigma_dep, graph=False)]
torch.cuda.synchronize()
tx, ty = W // 8, H // 4
cost = (A.view(H, W) > 0).view(ty, 4, tx, 8).sum(dim=(1, 3)).flatten()
orders = {"row-major": None,
          "costly first": torch.argsort(-cost.float(), stable=True).int(),
          "centre out": torch.argsort(((torch.arange(ty, device="cuda")[:, None] * 4 + 2 - H / 2) ** 2 +
                                       (torch.arange(tx, device="cuda")[None, :] * 8 + 4 - W / 2) ** 2)
                                      .flatten().float(), stable=True).int(),
          "costly last": torch.argsort(cost.float(), stable=True).int()}
yy = torch.arange(ty, device="cuda")[:, None].expand(ty, tx).flatten()
xx = torch.arange(tx, device="cuda")[None, :].expand(ty, tx).flatten()
cy_, cx_ = (yy * 4 + 2 - H / 2).float(), (xx * 8 + 4 - W / 2).float()
orders["centre out chebyshev"] = torch.argsort(torch.maximum(cy_.abs(), cx_.abs()), stable=True).int()
for bs in (2, 4, 8):  # blocks of bs x bs tiles, centre-out by block, row-major inside
    by, bx = yy // bs, xx // bs
    bc = ((by * bs * 4 + bs * 2 - H / 2) ** 2 + (bx * bs * 8 + bs * 4 - W / 2) ** 2).float()
    key = bc * 1e6 + ((yy % bs) * bs + xx % bs).float()
    orders[f"centre out {bs}x{bs} blocks"] = torch.argsort(key, stable=True).int()
def morton2(x, y):
    r = torch.zeros_like(x)
    for b in range(12):
        r |= ((x >> b) & 1) << (2 * b) | ((y >> b) & 1) << (2 * b + 1)
    return r
orders["morton"] = torch.argsort(morton2(xx, yy), stable=True).int()
cost_blk = torch.zeros(ty // 4 * (tx // 4), device="cuda").index_add_(0, (yy // 4) * (tx // 4) + xx // 4, cost.float())
key = -cost_blk[(yy // 4) * (tx // 4) + xx // 4] * 1e6 + ((yy % 4) * 4 + xx % 4).float()
orders["costly 4x4 blocks first"] = torch.argsort(key, stable=True).int()
for name, o in orders.items():
    fn(None if o is None else C.c_void_p(o.contiguous().data_ptr()))
    t = render()
    F2, A2, D2 = fp.run(pose, cam, lambda_th=sc.lambda_th, sigma_dep=sc.sigma_dep, graph=False)
    torch.cuda.synchronize()
    print(f"{name:14s} render {t:.4f} ms  same F {bool(torch.equal(F, F2))}")
