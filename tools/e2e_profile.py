#!/usr/bin/env python3
"""C3 through the host API (pinned buffers) with per-kernel CUDA events on: wall time of the call against the sum of
the kernels' times (how busy the GPU is while the rolling / chunked host solve runs).  Env knobs as the library's."""
import ctypes
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2203_11154_b200 as P  # noqa: E402
from paper_2203_11154_b200 import _native as N  # noqa: E402

n, S = 512, int(os.environ.get("SHIFTS", "256"))
cfg = P.MultigridConfig(P.CycleKind.V, 2, 2, 4, 1e-10, 200, P.SmootherConfig.vanka())
lams = P.circulant_shifts(1e-3, 256, 1 / 256, 0, S)
b = P.random_rhs(n, 2, count=S)
with P.BatchedMultigridHierarchy(P.Grid2D(n), lams, cfg) as H:
    nbytes = b.nbytes
    hb, hu = N.lib().pdmg_host_alloc(nbytes), N.lib().pdmg_host_alloc(nbytes)
    ctypes.memmove(hb, b.ctypes.data, nbytes)
    rep = N.SolveReport(0, 0, 0, 0, 0.0)
    for prof in (0, 1):
        N.lib().pdmg_solve(H._h, hb, hu, ctypes.byref(rep))
        H.set_profiling(bool(prof))
        N.lib().pdmg_reset_stats(H._h)
        t0 = time.perf_counter()
        for _ in range(3):
            assert N.lib().pdmg_solve(H._h, hb, hu, ctypes.byref(rep)) == 0
        wall = (time.perf_counter() - t0) / 3 * 1e3
        if prof:
            st = H.kernel_stats()
            tot = sum(v["ms"] for v in st.values()) / 3
            print(f"profiled: wall {wall:.2f} ms/solve, kernels {tot:.2f} ms/solve")
            for k, v in sorted(st.items(), key=lambda kv: -kv[1]["ms"]):
                print(f"   {k:36s} {v['launches'] // 3:5d} x {v['ms'] / max(v['launches'], 1) * 1e3:8.1f} us = {v['ms'] / 3:7.2f} ms")
        else:
            print(f"plain: wall {wall:.2f} ms/solve")
    N.lib().pdmg_host_free(hb)
    N.lib().pdmg_host_free(hu)
