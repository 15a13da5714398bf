"""Build libartemis tuning variants into variants/ (git-ignored)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2202_05628_b200 import build_lib  # noqa: E402

VARIANTS = {
    "base": (),
    "s24q8": ("ARTEMIS_SMEM_STACK=24",),
    "s24q6": ("ARTEMIS_SMEM_STACK=24", "ARTEMIS_QCAP=6", "ARTEMIS_QTHRESH=64"),
    "s24q6b4": ("ARTEMIS_SMEM_STACK=24", "ARTEMIS_QCAP=6", "ARTEMIS_QTHRESH=64",
                "ARTEMIS_MIN_BLOCKS=4"),
    "s28q6b4": ("ARTEMIS_SMEM_STACK=28", "ARTEMIS_QCAP=6", "ARTEMIS_QTHRESH=64",
                "ARTEMIS_MIN_BLOCKS=4"),
    "s24q5b4": ("ARTEMIS_SMEM_STACK=24", "ARTEMIS_QCAP=5", "ARTEMIS_QTHRESH=48",
                "ARTEMIS_MIN_BLOCKS=4"),
    "s24q8t96": ("ARTEMIS_SMEM_STACK=24", "ARTEMIS_QTHRESH=96"),
}
names = sys.argv[1:] or list(VARIANTS)
repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for n in names:
    out = os.path.join(repo, "variants", f"libartemis_{n}.so")
    build_lib.build(force=True, out=out, defines=VARIANTS[n])
    print(n, out)
