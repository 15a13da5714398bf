"""Build libartemis tuning variants into variants/ (git-ignored)."""
import itertools
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2202_05628_b200 import build_lib  # noqa: E402

VARIANTS = {
    "base": (),
    "q4": ("ARTEMIS_QCAP=4", "ARTEMIS_QTHRESH=48"),
    "q4s24": ("ARTEMIS_QCAP=4", "ARTEMIS_QTHRESH=48", "ARTEMIS_SMEM_STACK=24"),
    "q4s24b5": ("ARTEMIS_QCAP=4", "ARTEMIS_QTHRESH=48", "ARTEMIS_SMEM_STACK=24",
                "ARTEMIS_MIN_BLOCKS=5"),
    "q6t96": ("ARTEMIS_QCAP=6", "ARTEMIS_QTHRESH=96"),
    "q8t128": ("ARTEMIS_QCAP=8", "ARTEMIS_QTHRESH=128"),
    "q8t32": ("ARTEMIS_QCAP=8", "ARTEMIS_QTHRESH=32"),
}
names = sys.argv[1:] or list(VARIANTS)
repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for n in names:
    out = os.path.join(repo, "variants", f"libartemis_{n}.so")
    build_lib.build(force=True, out=out, defines=VARIANTS[n])
    print(n, out)
