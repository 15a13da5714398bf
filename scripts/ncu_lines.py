"""Per-CUDA-source-line stall samples and executed instructions from an ncu report."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
cur_file = ""
agg = {}
hdr = None
line_src = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0]:  # a source line row (aggregated metrics)
        key = (cur_file, int(r[0]))
        line_src[key] = r[1].strip()
        def num(v):
            try:
                return int(v.replace(",", ""))
            except ValueError:
                return 0
        stall = num(r[4])
        inst = num(r[7])
        a = agg.setdefault(key, [0, 0])
        a[0] += stall
        a[1] += inst
tot_s = sum(v[0] for v in agg.values()) or 1
tot_i = sum(v[1] for v in agg.values()) or 1
print(f"total stall samples {tot_s}, warp instructions {tot_i}")
for key, (st, ins) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{key[0]}:{key[1]:<5} stall {st / tot_s * 100:5.1f}%  inst {ins / tot_i * 100:5.1f}%  {line_src[key][:70]}")
