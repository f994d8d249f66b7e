#!/usr/bin/env python3
"""Summarize one ncu --set full capture exported by tools/ncu_top.sh (<tag>_raw.csv, <tag>_sass.csv.gz):
key counters, stall-reason totals from the source page, and the executed instruction mix.
    python tools/ncu_summary.py gpurun_out/<tag> "<title line>" > profiles/<name>_summary.txt"""
import collections
import csv
import gzip
import sys

tag, title = sys.argv[1], sys.argv[2]
rows = list(csv.reader(open(tag + "_raw.csv")))
hdr, units, r = rows[0], rows[1], rows[2]
print(title)
for w in ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
          "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
          "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
          "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__block_size",
          "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]:
    if w in hdr:
        i = hdr.index(w)
        print(f"  {w:64s} {r[i]} {units[i]}")
try:
    srows = list(csv.reader(gzip.open(tag + "_sass.csv.gz", "rt")))
except OSError:
    sys.exit(0)
k = next(i for i, x in enumerate(srows) if x and x[0] == "Address")
sh, data = srows[k], srows[k + 1:]
ix = {h: i for i, h in enumerate(sh)}
num = lambda x: float(x) if x.replace(".", "", 1).isdigit() else 0.0  # noqa: E731
stalls = collections.Counter()
for h in sh:
    if h.startswith("stall_") and "(Not Issued)" not in h:
        stalls[h] = sum(num(d[ix[h]]) for d in data)
tot = sum(stalls.values()) or 1
print("  stall samples (ncu source page, all samples):")
for h, v in stalls.most_common(8):
    print(f"    {h:26s} {int(v):8d} {v / tot:.3f}")
mix = collections.Counter()
for d in data:
    t = d[ix["Source"]].split()
    if t:
        op = t[1] if t[0].startswith("@") else t[0]
        mix[op.split(".")[0]] += num(d[ix["Instructions Executed"]])
tm = sum(mix.values()) or 1
print("  executed instruction mix (warp-level):")
for op, v in mix.most_common(12):
    print(f"    {op:10s} {v / tm:.3f}")
