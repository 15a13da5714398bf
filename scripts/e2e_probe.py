"""Host-side cost breakdown of the end-to-end frame stream (GPU box)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2202_05628_b200 import kinematics as KM  # noqa: E402
from paper_2202_05628_b200 import synthetic as S  # noqa: E402
from paper_2202_05628_b200.frame import FramePipeline  # noqa: E402

sc = S.make_scene("c3", frames=24)
fp = FramePipeline.from_scene(sc)
items = [(KM.PoseSpec.make(sc.poses[f]), sc.cameras[f][0]) for f in range(24)]


def timeit(fn, n=20):
    fn()
    t = time.perf_counter()
    for _ in range(n):
        fn()
    return (time.perf_counter() - t) / n * 1e3


print("pose_tables ms", timeit(lambda: fp.tables(items[3][0])))
print("camera ms", timeit(lambda: fp.camera(items[3][1])))
for readout in ("box", "records", "dense"):
    for _ in fp.run_stream(items[:4], readout=readout):
        pass
    torch.cuda.synchronize()
    t = time.perf_counter()
    n = 0
    for _ in fp.run_stream(items, readout=readout):
        n += 1
    dt = (time.perf_counter() - t) / n * 1e3
    print(f"run_stream readout={readout}: {dt:.3f} ms/frame, d2h MB/frame "
          f"{np.mean(getattr(fp, 'last_stream_d2h_bytes', [0])) / 1e6:.1f}")
# GPU-only frame time (graph replay, no readout)
cams = [fp.camera(c) for _, c in items]
tabs = [fp.tables(p) for p, _ in items]
fp.run(items[0][0], cams[0], tables=tabs[0])
torch.cuda.synchronize()
t = time.perf_counter()
for i in range(24):
    fp.run(items[i][0], cams[i], tables=tabs[i])
torch.cuda.synchronize()
print("graph frames only ms", (time.perf_counter() - t) / 24 * 1e3)
t = time.perf_counter()
for i in range(24):
    fp.run(items[i][0], items[i][1])
torch.cuda.synchronize()
print("frames incl host FK+camera ms", (time.perf_counter() - t) / 24 * 1e3)
