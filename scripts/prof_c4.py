"""One c4 stereo frame (warp + rebuild once, two eyes), eager, for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2202_05628_b200 import kinematics as KM  # noqa: E402
from paper_2202_05628_b200 import synthetic as S  # noqa: E402
from paper_2202_05628_b200.frame import FramePipeline  # noqa: E402

sc = S.make_scene("c4", frames=2)
fp = FramePipeline.from_scene(sc)
for f in range(2):
    pose = KM.PoseSpec.make(sc.poses[f])
    for i, cam in enumerate(sc.cameras[f]):
        fp.run(pose, cam, lambda_th=sc.lambda_th, sigma_dep=sc.sigma_dep, graph=False,
               reuse_tree=i > 0)
torch.cuda.synchronize()
print("ok")
