"""Per-kernel table (time, HBM GB/s vs peak, L2 hit rate, L2 bytes) from an
ncu --metrics CSV of scripts/prof_frame.py (last frame in the capture)."""
import collections
import csv
import json
import os
import sys

path = sys.argv[1]
peak = 6459.9
mp = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                  "MEASURED_PEAKS.json")
if os.path.exists(mp):
    peak = json.load(open(mp))["hbm_gbs"]
rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
hdr, rows = rows[0], rows[1:]
ix = {k: i for i, k in enumerate(hdr)}
launch = collections.OrderedDict()
for r in rows:
    d = launch.setdefault(int(r[ix["ID"]]), {"name": r[ix["Kernel Name"]].split("(")[0]})
    v = r[ix["Metric Value"]].replace(",", "")
    unit = r[ix["Metric Unit"]]
    try:
        x = float(v)
    except ValueError:
        continue
    scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "usecond": 1e-6,
             "nsecond": 1e-9, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6,
             "ms": 1e-3, "s": 1.0, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1.0)
    d[r[ix["Metric Name"]]] = x * scale
frames, cur = [], []
for d in launch.values():
    if d["name"].startswith("void lbs_warp_kernel") and cur:
        frames.append(cur)
        cur = []
    cur.append(d)
frames.append(cur)
last = frames[-1]
tot = sum(k["gpu__time_duration.sum"] for k in last)
print(f"# last captured frame: {len(last)} launches, {tot * 1e6:.1f} us (cold, serialised; "
      f"HBM peak {peak} GB/s measured)")
print(f"{'kernel':<44} {'us':>8} {'share':>6} {'HBM GB/s':>9} {'of peak':>8} {'L2 hit':>7} "
      f"{'DRAM MB':>8} {'L2 MB':>8}")
for k in last:
    t = k["gpu__time_duration.sum"]
    dram = k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0)
    gbs = dram / t / 1e9 if t else 0.0
    name = k["name"][5:] if k["name"].startswith("void ") else k["name"]
    print(f"{name[:44]:<44} {t * 1e6:8.1f} {100 * t / tot:5.1f}% {gbs:9.0f} "
          f"{100 * gbs / peak:7.1f}% {k.get('lts__t_sector_hit_rate.pct', 0):6.1f}% "
          f"{dram / 1e6:8.1f} {k.get('lts__t_bytes.sum', 0) / 1e6:8.1f}")
