"""Kernel timeline of graph-replayed frames (torch.profiler / CUPTI activity
records: device start/end of every kernel and memset inside the graph), to
see the gaps between the frame's stages. Prints one frame's records.

    python scripts/timeline.py [c2|c4|c1] [frames]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2202_05628_b200 import kinematics as KM  # noqa: E402
from paper_2202_05628_b200 import synthetic as S  # noqa: E402
from paper_2202_05628_b200.frame import FramePipeline  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 6
sc = S.make_scene("c3" if name == "c2" else name, frames=frames)
fp = FramePipeline.from_scene(sc)
poses = [KM.PoseSpec.make(sc.poses[f]) for f in range(frames)]
tabs = [fp.tables(p) for p in poses]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for f in range(2):
    fp.run(poses[f], sc.cameras[f][0], tables=tabs[f])
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for f in range(frames):
        with torch.cuda.stream(fp.stream):
            flush.fill_(f & 0xFF)
        fp.run(poses[f], sc.cameras[f][0], tables=tabs[f])
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
# frames are separated by the flush kernel (fill_)
groups, cur = [], []
for e in evs:
    if "fill" in e.name.lower() or "FillFunctor" in e.name:
        if cur:
            groups.append(cur)
        cur = []
        continue
    cur.append(e)
if cur:
    groups.append(cur)
for g in groups[-3:]:
    t0 = g[0].time_range.start
    print(f"--- frame: {len(g)} records, span {(g[-1].time_range.end - t0):.1f} us")
    prev_end = t0
    for e in g:
        s, en = e.time_range.start - t0, e.time_range.end - t0
        print(f"{s:9.1f} {en:9.1f} {en - s:8.1f}  gap {e.time_range.start - prev_end:7.1f}  {e.name[:70]}")
        prev_end = max(prev_end, e.time_range.end)
