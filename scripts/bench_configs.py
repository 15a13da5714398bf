"""Device time of every BASELINE config on one GPU (graph replay, CUDA
events on the pipeline stream, L2 flushed between steps), one JSON line per
config. A step is: c0 one 256^2 frame; c1 one pose rendered from 8 views of
512^2 (one warp + rebuild, 8 renders); c2 one 1024^2 frame; c3 the 64-frame
1024^2 sequence (reported per frame); c4 one stereo frame (one warp +
rebuild, two 1440x1600 eyes) on the ~4M-leaf, 32-joint asset.

    python scripts/bench_configs.py [c0 c1 c2 c3 c4] [--steps K]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2202_05628_b200 import kinematics as KM  # noqa: E402
from paper_2202_05628_b200 import synthetic as S  # noqa: E402
from paper_2202_05628_b200.frame import FramePipeline  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
steps = 10
for a in sys.argv[1:]:
    if a.startswith("--steps="):
        steps = int(a.split("=")[1])
names = args or ["c0", "c1", "c2", "c3", "c4"]
if os.environ.get("ARTEMIS_RENDER_BLOCKS"):  # experiment: cap the persistent render grid
    from paper_2202_05628_b200 import _lib  # noqa: E402
    _lib.lib().artemis_debug_set_render_blocks(int(os.environ["ARTEMIS_RENDER_BLOCKS"]))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

for name in names:
    t0 = time.time()
    frames = 64 if name == "c3" else max(steps + 3, 4)
    sc = S.make_scene(name, frames=frames)
    frames = len(sc.poses)
    fp = FramePipeline.from_scene(sc)
    gen_s = time.time() - t0
    st = fp.stream
    n_steps = 64 if name == "c3" else steps
    tabs = [KM.pose_tables(sc.rig, KM.PoseSpec.make(sc.poses[f])) for f in range(frames)]
    cams = [[fp.camera(c) for c in sc.cameras[f]] for f in range(frames)]

    sep = os.environ.get("ARTEMIS_VIEWS_SEPARATE") == "1"  # one render launch per view

    def step(f):
        pose = KM.PoseSpec.make(sc.poses[f])
        if len(cams[f]) > 1 and not sep:  # all views of the pose in one render launch
            fp.run_views(pose, cams[f], lambda_th=sc.lambda_th, sigma_dep=sc.sigma_dep,
                         tables=tabs[f])
            return
        for v, cam in enumerate(cams[f]):
            fp.run(pose, cam, lambda_th=sc.lambda_th, sigma_dep=sc.sigma_dep, tables=tabs[f],
                   reuse_tree=v > 0)

    for f in range(6):  # warm-up under the timed conditions (L2 flushed before each step)
        with torch.cuda.stream(st):
            flush.fill_(f & 0xFF)
        step(f % frames)
    st.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(n_steps)]
    for s in range(n_steps):
        f = s % frames
        with torch.cuda.stream(st):
            flush.fill_(s & 0xFF)
        ev[s][0].record(st)
        step(f)
        ev[s][1].record(st)
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in ev) / n_steps
    views = len(sc.cameras[0])
    W, H = sc.cameras[0][0].width, sc.cameras[0][0].height
    rays = views * W * H
    n_in, n_live = fp.counts()
    print(json.dumps({"config": name, "ms_per_step": ms, "rays_per_step": rays,
                      "rays_per_s": rays / (ms / 1e3), "views_per_step": views,
                      "image": [W, H], "voxels": sc.n_voxels, "live_leaves": n_live,
                      "channels": sc.channels, "joints": sc.rig.n_joints, "steps": n_steps,
                      "scene_gen_s": round(gen_s, 1)}), flush=True)
    fp.close()
    del fp, sc
    torch.cuda.empty_cache()
