"""Build libartemis tuning variants into variants/ (git-ignored)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2202_05628_b200 import build_lib  # noqa: E402

VARIANTS = {
    "base": (),
    "checks": ("ARTEMIS_DEBUG_CHECKS=1",),
    "sout": ("ARTEMIS_STREAM_OUT=1",),
    "flat": ("ARTEMIS_FLAT_SHADE=1",),
    "nocull": ("ARTEMIS_CULL=0",),
    "rcp": ("ARTEMIS_RCP_CROSSING=1",),
    "norcp": ("ARTEMIS_RCP_CROSSING=0", "ARTEMIS_FAST_CAMRAY=0"),
    "slowcam": ("ARTEMIS_FAST_CAMRAY=0",),
    "nopf": ("ARTEMIS_ROW_PREFETCH=0",),
    "pfl1": ("ARTEMIS_ROW_PREFETCH=3",),
    "smask": ("ARTEMIS_SMEM_MASK=1",),
    "ac2": ("ARTEMIS_A_CHECK=2",),
    "ac3": ("ARTEMIS_A_CHECK=3",),
    "ac2t40": ("ARTEMIS_A_CHECK=2", "ARTEMIS_QTHRESH=40"),
    "t40": ("ARTEMIS_QTHRESH=40",),
    "t56": ("ARTEMIS_QTHRESH=56",),
    "q4b5": ("ARTEMIS_QCAP=4", "ARTEMIS_QTHRESH=48", "ARTEMIS_MIN_BLOCKS=5"),
    "q4t40b5": ("ARTEMIS_QCAP=4", "ARTEMIS_QTHRESH=40", "ARTEMIS_MIN_BLOCKS=5"),
    "q4t56b5": ("ARTEMIS_QCAP=4", "ARTEMIS_QTHRESH=56", "ARTEMIS_MIN_BLOCKS=5"),
    "flat_nopf": ("ARTEMIS_FLAT_SHADE=1", "ARTEMIS_ROW_PREFETCH=0"),
    "rhint": ("ARTEMIS_ROW_HINT=1",),
    "sout_rhint": ("ARTEMIS_STREAM_OUT=1", "ARTEMIS_ROW_HINT=1"),
    "sout_nopf": ("ARTEMIS_STREAM_OUT=1", "ARTEMIS_ROW_PREFETCH=0"),
    "clocks": ("ARTEMIS_PHASE_CLOCKS=1",),
    "nodedup": ("ARTEMIS_DEDUP=0",),
    "q8t96": ("ARTEMIS_QCAP=8", "ARTEMIS_QTHRESH=96", "ARTEMIS_MIN_BLOCKS=3"),
    "q4t48": ("ARTEMIS_QCAP=4", "ARTEMIS_QTHRESH=48"),
    "b3": ("ARTEMIS_MIN_BLOCKS=3",),
    "b5": ("ARTEMIS_MIN_BLOCKS=5",),
    "noshade": ("ARTEMIS_NOSHADE=1",),
    "q5t56": ("ARTEMIS_QCAP=5", "ARTEMIS_QTHRESH=56"),
    "q5t64": ("ARTEMIS_QCAP=5", "ARTEMIS_QTHRESH=64"),
    "q4t48b": ("ARTEMIS_QCAP=4", "ARTEMIS_QTHRESH=48"),
    "noshade_nopf": ("ARTEMIS_NOSHADE=1", "ARTEMIS_ROW_PREFETCH=0"),
    "pf1": ("ARTEMIS_ROW_PREFETCH=2",),
    "q8": ("ARTEMIS_QCAP=8", "ARTEMIS_QTHRESH=96"),
    "t48": ("ARTEMIS_QTHRESH=48",),
    "b6": ("ARTEMIS_MIN_BLOCKS=6",),
    "t96": ("ARTEMIS_QTHRESH=96",),
    "t32": ("ARTEMIS_QTHRESH=32",),
    "q5t48": ("ARTEMIS_QCAP=5", "ARTEMIS_QTHRESH=48"),
    "q5t40": ("ARTEMIS_QCAP=5", "ARTEMIS_QTHRESH=40"),
    "q5t44": ("ARTEMIS_QCAP=5", "ARTEMIS_QTHRESH=44"),
    "q5t56": ("ARTEMIS_QCAP=5", "ARTEMIS_QTHRESH=56"),
    "t64": ("ARTEMIS_QTHRESH=64",),
    "bpf": ("ARTEMIS_ROW_PREFETCH=4",),
    "nosort": ("ARTEMIS_SORT_ITEMS=0",),
    "sortall": ("ARTEMIS_SORT_ITEMS=2",),
    "split2all": ("ARTEMIS_SPLIT_ALL=1",),
    "split3": ("ARTEMIS_SPLIT_M=3",),
    "nosplit": ("ARTEMIS_SPLIT_M=0",),
}
names = sys.argv[1:] or list(VARIANTS)
repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for n in names:
    out = os.path.join(repo, "variants", f"libartemis_{n}.so")
    build_lib.build(force=True, out=out, defines=VARIANTS[n])
    print(n, out)
