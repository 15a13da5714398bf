"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): every hot-path kernel at configs[0] size.

  camera mode  FramePipeline frames (warp -> onesweep sort -> resolve ->
               Karras build + brick map -> render_kernel<camera>), eager
  API mode     kernels.render_rays / forward_fit (render_kernel<kRender>,
               <kTrace>, <kCount>) on the brick walk and on the tree DFS
  sort         kernels.sort_order on 32- and 64-bit keys (onesweep,
               decoupled look-back)
  resolve      pipeline.resolve_collisions with heavy collisions
"""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_2202_05628_b200 import kernels as K  # noqa: E402
from paper_2202_05628_b200 import kinematics as KM  # noqa: E402
from paper_2202_05628_b200 import pipeline as P  # noqa: E402
from paper_2202_05628_b200 import synthetic as S  # noqa: E402
from paper_2202_05628_b200 import types as T  # noqa: E402
from paper_2202_05628_b200.frame import FramePipeline  # noqa: E402

sc = S.make_scene("c0", frames=2, image=(128, 96))
fp = FramePipeline.from_scene(sc)
for f in range(2):
    fp.run(KM.PoseSpec.make(sc.poses[f]), sc.cameras[f][0], graph=False, parity=True,
           lambda_th=sc.lambda_th, sigma_dep=sc.sigma_dep)
torch.cuda.synchronize()
t = fp.tree()
fp.close()

pose = KM.PoseSpec.make(sc.poses[0])
tables = KM.pose_tables(sc.rig, pose)
cam = sc.cameras[0][0]
R, origin = cam.cam_to_world()
og, dg, dw = oracle.camera_rays(R, origin, cam.fx, cam.fy, cam.cx, cam.cy, cam.width,
                                cam.height, sc.lo, sc.cell_size)
tree = (t["codes"], t["flut_idx"], t["root"], t["left"], t["right"], t["box_min"],
        t["box_size"])
for mode in ("walk", "dfs"):
    K.DeviceTree.MAX_BRICK_TABLE = 0 if mode == "dfs" else 1 << 24
    K.invalidate_cache()
    args = (*tree, og, dg, dw, 0.0, np.inf, sc.flut32, t["rotation_joint"], tables.rot_inv,
            sc.degree, sc.channels)
    K.render_rays(*args, sc.lambda_th, sc.sigma_dep, True)
    K.forward_fit(*args)
    K.traverse_ray(*tree, og[5000], dg[5000], 0.0, np.inf)
torch.cuda.synchronize()

rng = np.random.default_rng(0)
K.sort_order(rng.integers(0, 1 << 30, size=300_001).astype(np.uint64))
K.sort_order(rng.integers(0, 1 << 62, size=100_003).astype(np.uint64))

n = 20_000
cells = (1 + rng.integers(0, 8, size=(n, 3))).astype(np.int32)
sigma = np.round(rng.uniform(0, 3, n), 1)
warp = T.WarpResult(16, np.zeros(3), np.full(3, 1 / 16), np.zeros((n, 3)), cells,
                    np.zeros((n, 4)), np.zeros(n, np.int32), np.eye(3)[None], np.ones(n, bool),
                    ())


class F:
    densities = sigma


P.resolve_collisions(warp, F)
torch.cuda.synchronize()
print("sanitize target ok")
