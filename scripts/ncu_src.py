"""Per-source-line totals (instructions executed, stall samples) from an ncu
report's `--page source --print-source cuda,sass` view."""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout.splitlines()
cur = ""
hdr = None
agg = collections.defaultdict(lambda: [0, 0, ""])
line = None
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
    if r[0]:  # a source line row (then its SASS rows follow with empty line no)
        line = (cur, int(r[0]))
        agg[line][2] = r[1].strip()[:70]
    d = dict(zip(hdr[2:], r[2:]))
    try:
        agg[line][0] += int(d.get("Instructions Executed", "0") or 0)
        agg[line][1] += int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
    except (ValueError, TypeError):
        pass
tot_i = sum(v[0] for v in agg.values()) or 1
tot_s = sum(v[1] for v in agg.values()) or 1
print(f"total warp instructions {tot_i}, stall samples {tot_s}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{k[0]}:{k[1]:<5} inst {100 * v[0] / tot_i:5.1f}%  stall {100 * v[1] / tot_s:5.1f}%  {v[2]}")
