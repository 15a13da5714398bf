"""Render c2 frames with the phase-clock variant and print the phase split."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2202_05628_b200 import _lib  # noqa: E402
from paper_2202_05628_b200 import kinematics as KM  # noqa: E402
from paper_2202_05628_b200 import synthetic as S  # noqa: E402
from paper_2202_05628_b200.frame import FramePipeline  # noqa: E402

sc = S.make_scene("c3", frames=3)
fp = FramePipeline.from_scene(sc)
L = _lib.load_library()
fn = L.artemis_debug_phase_clocks
fn.argtypes = [C.c_void_p, C.c_int]
buf = (C.c_ulonglong * 17)()
for f in range(3):
    fp.run(KM.PoseSpec.make(sc.poses[f]), sc.cameras[f][0], graph=False)
    torch.cuda.synchronize()
    fn(C.addressof(buf), 1)
vals = list(buf)[:7]
fb, tests = buf[7], buf[8]
print(f"box tests {tests} exact fallbacks {fb} ({fb / max(tests, 1) * 100:.3f}%)")
print(f"walk: crossings {buf[9]} cell steps {buf[10]} brick skips {buf[11]} axis syncs {buf[12]}")
print(f"shade: visible entries {buf[13]} same-level groups {buf[14]} warp-round unique rows "
      f"{buf[15]} rounds {buf[16]} (reuse same-level {buf[13] / max(buf[14], 1):.2f}x, "
      f"warp-round {buf[13] / max(buf[15], 1):.2f}x)")
tot = sum(vals)
names = ["refill", "A traverse", "B1 exact", "B2 chain", "C shade", "retire", "tail"]
print(" ".join(f"{n}={v / tot * 100:.1f}%" for n, v in zip(names, vals)))
