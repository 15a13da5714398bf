"""Hit statistics per config (first frame / view): rays, hit rays, hits."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2202_05628_b200 import kernels as K  # noqa: E402
from paper_2202_05628_b200 import kinematics as KM  # noqa: E402
from paper_2202_05628_b200 import synthetic as S  # noqa: E402
from paper_2202_05628_b200.frame import FramePipeline  # noqa: E402

for name in sys.argv[1:] or ["c0", "c1", "c2", "c4"]:
    sc = S.make_scene(name, frames=1)
    fp = FramePipeline.from_scene(sc)
    pose = KM.PoseSpec.make(sc.poses[0])
    fp.run(pose, sc.cameras[0][0], graph=False, parity=True)
    tree = fp.tree()
    shade = K.DeviceShading(np.zeros((sc.n_voxels, 2)), np.zeros(sc.n_voxels, np.int32),
                            np.eye(3)[None], 0, 1)
    dtree = K.DeviceTree(tree["codes"], tree["flut_idx"], tree["root"], tree["left"],
                         tree["right"], tree["box_min"], tree["box_size"], shade)
    cam = sc.cameras[0][0]
    R, origin = cam.cam_to_world()
    og, dg, dw = K.camera_rays_device(R, origin, cam.fx, cam.fy, cam.cx, cam.cy, cam.width,
                                      cam.height, sc.lo, sc.cell_size)
    counts = K.count_hits_device(dtree, K.DeviceRays.from_tensors(og, dg, dw))
    n = cam.width * cam.height
    hr = int((counts > 0).sum())
    h = int(counts.sum())
    print(f"{name}: rays {n} hit rays {hr} ({hr / n:.1%}) hits {h} hits/hit-ray {h / max(hr, 1):.1f} "
          f"leaves {tree['n_live']} FLUT MB {sc.flut32.nbytes / 1e6:.0f}", flush=True)
    fp.close()
    del dtree, counts
    torch.cuda.empty_cache()
