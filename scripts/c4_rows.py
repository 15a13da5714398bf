"""configs[4]: FLUT rows each eye's render touches (unique leaves hit by the
eye's rays, from the device hit trace) -> compulsory row bytes, to compare
with the ncu DRAM bytes of the eye's render launch."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2202_05628_b200 import kernels as K  # noqa: E402
from paper_2202_05628_b200 import kinematics as KM  # noqa: E402
from paper_2202_05628_b200 import synthetic as S  # noqa: E402
from paper_2202_05628_b200.frame import FramePipeline  # noqa: E402

sc = S.make_scene("c4", frames=1)
fp = FramePipeline.from_scene(sc)
pose = KM.PoseSpec.make(sc.poses[0])
fp.run(pose, sc.cameras[0][0], graph=False, parity=True)
torch.cuda.synchronize()
t = fp.tree()
shade = K.DeviceShading(np.zeros((sc.n_voxels, 2)), np.zeros(sc.n_voxels, np.int32),
                        np.eye(3)[None], 0, 1)
tree = K.DeviceTree(t["codes"], t["flut_idx"], t["root"], t["left"], t["right"], t["box_min"],
                    t["box_size"], shade)
out = {"live_leaves": int(t["n_live"])}
rows_all = []
for e, cam in enumerate(sc.cameras[0]):
    R, origin = cam.cam_to_world()
    og, dg, dw = K.camera_rays_device(R, origin, cam.fx, cam.fy, cam.cx, cam.cy, cam.width,
                                      cam.height, sc.lo, sc.cell_size)
    rays = K.DeviceRays.from_tensors(og, dg, dw)
    _, _, off, hidx, _, _ = K.forward_fit_device(tree, shade, rays)
    u = torch.unique(hidx)
    rows_all.append(u)
    out[f"eye{e}"] = {"rays": cam.width * cam.height, "hits": int(hidx.numel()),
                      "hit_rays": int((np.diff(off) > 0).sum()), "unique_rows": int(u.numel()),
                      "row_bytes_MB": int(u.numel()) * 9 * sc.channels * 4 / 1e6}
    del og, dg, dw, hidx, rays
out["union_rows"] = int(torch.unique(torch.cat(rows_all)).numel())
print(json.dumps(out))
