"""Per-launch table of an `ncu --metrics ... --csv --log-file X.csv` capture:
kernel, duration (us) and every other metric captured, one line per launch."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
launches = collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    key = d["ID"]
    e = launches.setdefault(key, {"name": d["Kernel Name"].split("(")[0][:48]})
    v = d["Metric Value"].replace(",", "")
    try:
        v = float(v)
    except ValueError:
        pass
    e[d["Metric Name"]] = v
for k, e in launches.items():
    dur = e.get("gpu__time_duration.sum", 0) / 1e3
    extra = []
    for m, lab, sc in (("dram__bytes_read.sum", "dramR MB", 1e6), ("dram__bytes_write.sum", "dramW MB", 1e6),
                       ("lts__t_bytes.sum", "L2 MB", 1e6), ("l1tex__t_sector_hit_rate.pct", "L1 hit%", 1),
                       ("smsp__inst_executed.sum", "Minst", 1e6)):
        if m in e:
            extra.append(f"{lab} {e[m] / sc:8.1f}")
    print(f"{k:>4} {e['name']:<48} {dur:9.1f} us  " + "  ".join(extra))
