"""Per-call overhead of the kernel-contract shim: one
integrate_ray-style call (render_rays on ONE ray, render.py:209-231) on the
configs[0] and configs[2] FLUTs, cold (first call: upload + split + tree
pack + brick map) and warm (device copies reused), under both cache
policies. Prints a small table for profiles/."""
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_2202_05628_b200 import kernels as K  # noqa: E402
from paper_2202_05628_b200 import kinematics as KM  # noqa: E402
from paper_2202_05628_b200 import synthetic as S  # noqa: E402

print(f"{'config':<8}{'FLUT':>10}{'policy':>10}{'cold ms':>10}{'warm ms (median of 50)':>24}"
      f"{'H2D per warm call':>20}")
for name in ("c0", "c2"):
    sc = S.make_scene(name)
    tables = KM.pose_tables(sc.rig, KM.PoseSpec.make(sc.poses[0]))
    fr = oracle.render_frame(sc, tables, sc.cameras[0][0], render=False,
                             flut64=sc.flut32[:, -1:].astype(np.float64))
    flut = sc.flut64()
    cnt = oracle.count_hits(*fr["tree"], fr["origins_g"], fr["dirs_g"], 0.0, np.inf)
    r = int(np.flatnonzero(cnt > 0)[len(np.flatnonzero(cnt > 0)) // 2])
    ray = (fr["origins_g"][r:r + 1], fr["dirs_g"][r:r + 1], fr["dirs_w"][r:r + 1])
    args = (*fr["tree"], *ray, 0.0, np.inf, flut, fr["rotation_joint"], tables.rot_inv,
            sc.degree, sc.channels, sc.lambda_th, sc.sigma_dep, True)
    for policy in ("content", "identity"):
        K.set_cache_policy(policy)
        torch.cuda.synchronize()
        t = time.perf_counter()
        K.render_rays(*args)
        cold = time.perf_counter() - t
        s0 = K.cache_stats()
        times = []
        for _ in range(50):
            t = time.perf_counter()
            K.render_rays(*args)
            times.append(time.perf_counter() - t)
        s1 = K.cache_stats()
        h2d = (s1["h2d_bytes"] - s0["h2d_bytes"]) / 50
        print(f"{name:<8}{flut.nbytes / 1e6:>8.0f}MB{policy:>10}{cold * 1e3:>10.1f}"
              f"{np.median(times) * 1e3:>24.2f}{h2d:>18.0f} B")
    K.set_cache_policy("content")
    del flut
