#!/usr/bin/env python3
"""Small cases that launch every kernel family of libpdmg_b200.so once or more -- the workload of the
compute-sanitizer runs recorded in profiles/ (one tool per gpurun call):
    compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck python tools/sanitize_cases.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2203_11154_b200 as P  # noqa: E402
from paper_2203_11154_b200 import lfa  # noqa: E402


def main():
    V = P.SmootherConfig.vanka()
    lams = P.circulant_shifts(0.01, 32, 1 / 32, 0, 3)
    # one-CTA-per-shift solve (k_small_solve), both precisions
    for prec in ("c128", "c64"):
        with P.BatchedMultigridHierarchy(P.Grid2D(64), lams, P.MultigridConfig(P.CycleKind.V, 1, 1, 4, 1e-8, 30, V),
                                         precision=prec) as H:
            H.solve(P.random_rhs(64, 1, count=3))
    # batched level passes: k_march2 (two- and one-sweep, ragged strips), k_march (Jacobi), k_level, k_resid_norm,
    # the coarse tail (k_small_cycle), k_coarse_solve, pack/unpack, finalize, copy_words
    for cfg in (P.MultigridConfig(P.CycleKind.V, 2, 2, 4, 1e-8, 20, V), P.MultigridConfig(P.CycleKind.W, 1, 1, 25, 1e-8, 20, V),
                P.MultigridConfig(P.CycleKind.V, 1, 1, 25, 1e-8, 20, P.SmootherConfig.jacobi())):
        for prec in ("c128", "c64"):
            n = 200 if cfg.coarsest_n == 25 else 256
            with P.BatchedMultigridHierarchy(P.Grid2D(n), lams, cfg, precision=prec) as H:
                H.set_solve_path("batched")
                b = P.random_rhs(n, 2, count=3)
                H.solve(b)
                m = n - 1
                H.apply_smoother(0, b, b)
                H.residual(0, b, b)
                H.restrict_full_weighting(0, b)
                H.prolong_bilinear(0, b[:, : (n // 2 - 1), : (n // 2 - 1)].copy())
                H.norm(0, b)
                H.cycle(b, b)
    with P.BatchedMultigridHierarchy(P.Grid2D(16), lams, P.MultigridConfig(coarsest_n=4)) as H:
        H.coarse_solve(P.random_rhs(4, 3, count=3))
    # device list (sharded context) and ParaDIAG (time DFT, time GEMM, residuals), one and two shards
    with P.BatchedMultigridHierarchy(P.Grid2D(64), lams, P.MultigridConfig(P.CycleKind.V, 1, 1, 4, 1e-8, 20, V),
                                     devices=[0, 0]) as H:
        H.solve(P.random_rhs(64, 4, count=3))
    cfg = P.MultigridConfig(P.CycleKind.V, 1, 1, 4, 1e-8, 30, V)
    f = P.random_rhs(32, 5, count=6)
    for devs in (None, [0, 0]):
        with P.ParadiagCirculant(32, 6, 0.01, 1 / 6, cfg, devices=devs) as pd:
            pd.run(f)
    td = P.TimeDiscretization(P.TimeSchemeKind.HeatBVM, 6, 1 / 6, 0.01)
    P.paradiag_solve(f, td, cfg, devices=[0, 0])
    # LFA kernels
    lfa.smoothing_factor(10 + 40j, 1 / 32, V, lfa.LFAConfig(16))
    lfa.smoothing_factor_bound(10 + 40j, 1 / 32, 0.96, lfa.LFAConfig(16))
    m = lfa.TwoGridModel(37j, 1 / 64, P.SmootherKind.Vanka, lfa.LFAConfig(16))
    m.rho([0.5, 0.9], 2)
    m.smoothing(0.9)
    lfa.optimize_omega(0.0, 1 / 64, P.SmootherKind.Jacobi, lfa.OmegaObjective.SmoothingMu, lfa=lfa.LFAConfig(16))
    print("sanitize cases ok")


if __name__ == "__main__":
    main()
