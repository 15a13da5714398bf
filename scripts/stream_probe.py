"""Timeline of FramePipeline.run_stream (box readout): per-frame device time
and the GPU idle gap before each frame, from CUDA events on the frame
stream; host time per stage of the loop."""
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
orig_run = FramePipeline.run
ev = []
host = []


def run(self, *a, **k):
    t0 = time.perf_counter()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(self.stream)
    out = orig_run(self, *a, **k)
    e1.record(self.stream)
    ev.append((e0, e1))
    host.append(time.perf_counter() - t0)
    return out


for _ in fp.run_stream(items[:4]):
    pass
torch.cuda.synchronize()
FramePipeline.run = run
t = time.perf_counter()
n = 0
for _ in fp.run_stream(items):
    n += 1
torch.cuda.synchronize()
wall = (time.perf_counter() - t) / n * 1e3
dev = [a.elapsed_time(b) for a, b in ev]
gaps = [ev[i - 1][1].elapsed_time(ev[i][0]) for i in range(1, len(ev))]
print(f"wall {wall:.3f} ms/frame; device per frame median {np.median(dev):.3f} ms; "
      f"gap before frame median {np.median(gaps):.3f} max {np.max(gaps):.3f} ms; "
      f"host run() median {np.median(host) * 1e3:.3f} ms")
