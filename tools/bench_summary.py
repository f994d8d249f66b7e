#!/usr/bin/env python3
"""One-line-per-kernel summary of bench.py JSON lines: bench_summary.py file.json [...]"""
import json
import sys

for p in sys.argv[1:]:
    try:
        d = json.loads(open(p).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(p, "unreadable:", e)
        continue
    par = d.get("parity") or {}
    e2e = d.get("e2e") or {}
    pg = d.get("e2e_pageable") or {}
    print(f"{p}: {d['ms_per_step']:.3f} ms/step  e2e {e2e.get('ms_per_step', float('nan')):.2f}  pageable "
          f"{pg.get('ms_per_step', float('nan')):.2f}  parity {par.get('iters_equal')} {par.get('max_rel_err_u')}")
    for k, v in (d.get("kernels") or {}).items():
        print(f"    {k:36s} {v['launches']:4d} x {v['ms'] / v['launches'] * 1000:8.1f} us   moved {v['moved_GBps']:7.1f} GB/s")
