"""Per-source-line executed warp instructions from an ncu report (sass rows
attributed to the preceding CUDA line), top lines and per-function-range sums."""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout.splitlines()
cur, hdr, line = "", None, None
agg = collections.Counter()
src = {}
for r in csv.reader(out):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "Function Name":
        continue
    if r[0]:
        line = (cur, int(r[0]))
        src[line] = r[1].strip()[:70]
    d = dict(zip(hdr[2:], r[2:]))
    try:
        agg[line] += int(d.get("Instructions Executed", "0") or 0)
    except ValueError:
        pass
tot = sum(agg.values())
print(f"total warp instructions {tot / 1e6:.1f} M")
for k, v in agg.most_common(top):
    if k is None:
        continue
    print(f"{k[0]}:{k[1]:<5} {v / 1e6:7.2f} M {100 * v / tot:5.1f}%  {src.get(k, '')}")
