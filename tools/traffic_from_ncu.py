#!/usr/bin/env python3
"""Stamp profiles/traffic.json with the ncu DRAM traffic of a kernel class from one `ncu --set full` capture.

    python tools/traffic_from_ncu.py <raw.csv from `ncu -i X.ncu-rep --page raw --csv`> <config> <kernel class> <source note>

Takes the mean of dram__bytes_read.sum + dram__bytes_write.sum over the captured launches and records it with the
sha256[:16] of the kernel sources in the tree (the build the capture must have profiled); bench.py reports the
figure only while that build is the one it runs.
"""
import csv
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    raw, config, kernel, note = sys.argv[1:5]
    rows = list(csv.reader(open(raw)))
    hdr = rows[0]
    units = rows[1]
    ir, iw = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    vals = []
    for r in rows[2:]:
        try:
            vals.append(float(r[ir].replace(",", "")) * scale[units[ir]] + float(r[iw].replace(",", "")) * scale[units[iw]])
        except (ValueError, KeyError, IndexError):
            pass
    if not vals:
        sys.exit("no dram__bytes rows in " + raw)
    sys.path.insert(0, ROOT)
    from paper_2203_11154_b200 import _native as N

    sha = N.source_sha16()
    p = os.path.join(ROOT, "profiles", "traffic.json")
    tj = json.load(open(p)) if os.path.exists(p) else {}
    tj.setdefault(config, {})[kernel] = {"bytes": sum(vals) / len(vals), "src_sha16": sha, "source": note,
                                         "launches_captured": len(vals)}
    json.dump(tj, open(p, "w"), indent=1)
    print(config, kernel, sum(vals) / len(vals), sha)


if __name__ == "__main__":
    main()
