"""Per-source-line stall-reason breakdown from an ncu report (sass rows
attributed to the preceding CUDA line in the cuda,sass source view)."""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
lo = int(sys.argv[3]) if len(sys.argv) > 3 else 0
hi = int(sys.argv[4]) if len(sys.argv) > 4 else 10 ** 9
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout.splitlines()
reasons = ["stall_long_sb", "stall_short_sb", "stall_wait", "stall_selected",
           "stall_branch_resolving", "stall_not_selected", "stall_no_inst", "stall_math",
           "stall_dispatch", "stall_mio", "stall_lg"]
cur = ""
hdr = None
agg = collections.defaultdict(lambda: collections.Counter())
src = {}
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
    if r[0]:
        line = (cur, int(r[0]))
        src[line] = r[1].strip()[:60]
    d = dict(zip(hdr[2:], r[2:]))
    for k in reasons + ["Instructions Executed"]:
        try:
            agg[line][k] += int(d.get(k, "0") or 0)
        except ValueError:
            pass
tot = collections.Counter()
for c in agg.values():
    tot.update(c)
sel = {k: v for k, v in agg.items() if k and lo <= k[1] <= hi}
S = sum(tot[r] for r in reasons) or 1
print("all-kernel stall shares:", {r[6:]: round(100 * tot[r] / S, 1) for r in reasons})
rows = sorted(sel.items(), key=lambda kv: -sum(kv[1][r] for r in reasons))[:top]
for k, c in rows:
    s = sum(c[r] for r in reasons)
    parts = ", ".join(f"{r[6:]} {100 * c[r] / S:.1f}" for r in reasons if c[r] > 0.05 * s)
    print(f"{k[0]}:{k[1]:<5} {100 * s / S:5.1f}%  [{parts}]  {src.get(k, '')}")
