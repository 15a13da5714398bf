"""configs[2] frame time with the configs' densities (no ray ever stops
early: alpha <= ~0.35) against an opaque body (densities x 64: the warp-level
early ray termination cuts the walk), lambda_th 1e-4 and 1e-12 (never stop).
Graph replay, L2 flushed between frames, CUDA events on the pipeline stream."""
import dataclasses
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2202_05628_b200 import kinematics as KM  # noqa: E402
from paper_2202_05628_b200 import synthetic as S  # noqa: E402
from paper_2202_05628_b200.frame import FramePipeline  # noqa: E402

base = S.make_scene("c2")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for gain in (1.0, 64.0):
    fl = base.flut32.copy()
    fl[:, -1] *= np.float32(gain)
    sc = dataclasses.replace(base, flut32=fl)
    fp = FramePipeline.from_scene(sc)
    pose, cam = KM.PoseSpec.make(sc.poses[0]), sc.cameras[0][0]
    for lam in (1e-4, 1e-12):
        ms = []
        for it in range(13):
            with torch.cuda.stream(fp.stream):
                flush.fill_(it)
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
            F, A, D = fp.run(pose, cam, graph=True, lambda_th=lam, sigma_dep=sc.sigma_dep)
            with torch.cuda.stream(fp.stream):
                e1.record()
            fp.stream.synchronize()
            if it >= 3:
                ms.append(e0.elapsed_time(e1))
        amax = float(A.max())
        print(f"density x{gain:g} lambda_th {lam:g}: frame {np.median(ms):.3f} ms "
              f"(min {min(ms):.3f}), max alpha {amax:.4f}")
    fp.close()
