"""Render a few eager frames of a config for ncu (one kernel per stage).

    python scripts/prof_frame.py [c2|c0|c4] [frames]

c4 renders both stereo eyes of each frame (run_views: one rebuild, one
render launch per eye for a FLUT beyond 16x L2)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2202_05628_b200 import kinematics as KM  # noqa: E402
from paper_2202_05628_b200 import synthetic as S  # noqa: E402
from paper_2202_05628_b200.frame import FramePipeline  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 3
if name == "c2":
    sc = S.make_scene("c3", frames=frames)
elif name == "c4":
    sc = S.make_scene("c4", frames=frames)
else:
    sc = S.make_scene("c0", frames=frames)
fp = FramePipeline.from_scene(sc)
for f in range(frames):
    pose = KM.PoseSpec.make(sc.poses[f])
    if name == "c4":
        fp.run_views(pose, sc.cameras[f], lambda_th=sc.lambda_th, sigma_dep=sc.sigma_dep,
                     graph=False)
    else:
        fp.run(pose, sc.cameras[f][0], lambda_th=sc.lambda_th, sigma_dep=sc.sigma_dep,
               graph=False)
torch.cuda.synchronize()
print("frames ok", fp.counts())
