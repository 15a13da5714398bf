"""Summarise an ncu --metrics gpu__time_duration.sum,dram__bytes_* CSV launch
list into per-frame per-kernel rows (time share, DRAM bytes)."""
import collections
import csv
import sys

path = sys.argv[1]
rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
hdr, rows = rows[0], rows[1:]
ix = {k: i for i, k in enumerate(hdr)}
launch = collections.OrderedDict()
for r in rows:
    d = launch.setdefault(int(r[ix["ID"]]), {"name": r[ix["Kernel Name"]].split("(")[0]})
    d[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
frames, cur = [], []
for lid, d in launch.items():
    name = d["name"].replace("artemis::", "")
    # a frame starts at its prepare kernel, or (older builds) at the warp kernel;
    # the bench's L2 flush (a torch fill kernel) starts a new step as well
    if cur and (name.startswith("frame_prepare_kernel") or "FillFunctor" in name or
                (name.startswith("void lbs_warp_kernel") and
                 not cur[-1]["name"].replace("artemis::", "").startswith("frame_prepare"))):
        frames.append(cur)
        cur = []
    cur.append(d)
frames.append(cur)
for f, ks in enumerate(frames):
    tot = sum(k["gpu__time_duration.sum"] for k in ks) / 1e3
    print(f"frame {f}: {len(ks)} launches, {tot:.1f} us total")
    for k in ks:
        t = k["gpu__time_duration.sum"] / 1e3
        print(f"  {k['name'].replace('artemis::', ''):<58} {t:9.1f} us {100 * t / tot:5.1f}%  dram rd "
              f"{k.get('dram__bytes_read.sum', 0) / 1e6:9.1f} MB wr "
              f"{k.get('dram__bytes_write.sum', 0) / 1e6:7.1f} MB")
