"""Summarise an ncu report: key section metrics, stall reasons, SASS hot spots."""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20


def run(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout


keys = ("Duration", "Elapsed Cycles", "DRAM Throughput", "L2 Hit Rate", "L1/TEX Hit Rate",
        "Executed Ipc Active", "Issue Slots Busy", "Achieved Active Warps Per SM",
        "Theoretical Active Warps per SM", "Registers Per Thread", "Avg. Active Threads Per Warp",
        "Executed Instructions", "Warp Cycles Per Issued Instruction", "Memory Throughput",
        "Dynamic Shared Memory Per Block", "Grid Size", "Eligible Warps Per Scheduler")
r = csv.reader(run("--page", "details", "--csv").splitlines())
hdr = next(r)
for row in r:
    d = dict(zip(hdr, row))
    if d.get("Metric Name") in keys:
        print(f"{d['Metric Name']:<40} {d['Metric Value']} {d['Metric Unit']}")
raw = run("--page", "raw", "--csv").splitlines()
rr = list(csv.reader(raw))
if len(rr) >= 3:
    names, vals = rr[0], rr[2]
    stall = {n: v for n, v in zip(names, vals) if n.startswith("smsp__average_warp_latency_issue_stalled") or n.startswith("smsp__warp_issue_stalled_") and n.endswith("_per_warp_active.pct")}
    items = []
    for n, v in stall.items():
        try:
            items.append((float(v.replace(",", "")), n))
        except ValueError:
            pass
    for v, n in sorted(items, reverse=True)[:12]:
        print(f"stall {n:<75} {v}")
    for n, v in zip(names, vals):
        if n in ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
                 "sm__warps_active.avg.pct_of_peak_sustained_active", "gpu__time_duration.sum"):
            print(f"{n:<60} {v}")
src = list(csv.reader(run("--page", "source", "--csv", "--print-source", "sass").splitlines()))
h = src[1]
rows = [dict(zip(h, x)) for x in src[2:]]
tot_s = sum(int(x["Warp Stall Sampling (All Samples)"]) for x in rows) or 1
tot_i = sum(int(x["Instructions Executed"]) for x in rows) or 1
op = collections.Counter()
for x in rows:
    t = x["Source"].split()
    o = (t[1] if t and t[0].startswith("@") and len(t) > 1 else (t[0] if t else "")).split(".")[0]
    op[o] += int(x["Instructions Executed"])
print("warp-instructions", tot_i)
print("mix", ", ".join(f"{k} {v / tot_i * 100:.1f}%" for k, v in op.most_common(14)))
for x in sorted(rows, key=lambda x: -int(x["Warp Stall Sampling (All Samples)"]))[:top]:
    print(f"{x['Address'][-5:]} {x['Source'][:58]:<58} stall={int(x['Warp Stall Sampling (All Samples)']) / tot_s * 100:5.1f}% n={x['Instructions Executed']} thr={x['Avg. Threads Executed']}")
