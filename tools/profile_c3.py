#!/usr/bin/env python3
"""One device-resident BASELINE config 3 solve (256 shifts, n = 512, V(2,2)) after one warm-up solve: the workload
the ncu captures in profiles/ are taken on (tools/ncu_top.sh).  --shifts / --config c4a / --nu as in bench.py."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2203_11154_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3", choices=["c3", "c4a", "c5solve"])
ap.add_argument("--shifts", type=int, default=0)
ap.add_argument("--precision", default="c128")
a = ap.parse_args()
n, S, alpha, nt, dt, seed, nu = {"c3": (512, 256, 1e-3, 256, 1 / 256, 2, 2), "c4a": (1024, 1024, 0.01, 1024, 1 / 1024, 3, 1),
                                  "c5solve": (256, 256, 0.01, 256, 1 / 256, 4, 1)}[a.config]
S = a.shifts or S
cfg = P.MultigridConfig(P.CycleKind.V, nu, nu, 4, 1e-5 if a.precision == "c64" else 1e-10, 200, P.SmootherConfig.vanka())
lams = P.circulant_shifts(alpha, nt, dt, 0, S)
b = P.random_rhs(n, seed, count=S)
d_b = torch.from_numpy(b.reshape(S, n - 1, n - 1).view(np.float64)).cuda()
d_u = torch.empty_like(d_b)
with P.BatchedMultigridHierarchy(P.Grid2D(n), lams, cfg, precision=a.precision) as H:
    for _ in range(2):
        reps = H.solve_device(d_b.data_ptr(), d_u.data_ptr())
    torch.cuda.synchronize()
print("cycles", sorted(set(r.iterations for r in reps)), "converged", all(r.converged for r in reps))
