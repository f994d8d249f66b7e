#!/usr/bin/env python3
"""Generate tests/golden/*.json from the REFERENCE's own code (TEST INFRASTRUCTURE).

Runs oracle/_ref/libpdmg_ref.so -- the reference's unmodified proj/src/grid.cpp + proj/src/smoother.cpp
compiled where they lie under /root/reference (oracle/Makefile), driven by the restated multigrid loop
(oracle/ref_driver.cpp) -- and writes small fixtures: RNG draws, operator outputs on small grids,
BASELINE config-1/2/3 solve results and the README W(1,0) rates.  The GPU box has no /root/reference,
so these committed fixtures are what pin the oracle there.

    make -C oracle && python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_lib import Cfg, Oracle, RefLib  # noqa: E402


def c2l(a):
    a = np.asarray(a, np.complex128).ravel()
    return [[float(z.real), float(z.imag)] for z in a]


def summary(u):
    u = np.asarray(u, np.complex128).ravel()
    return {"sum": c2l([u.sum()])[0], "sumsq": float(np.sum(np.abs(u) ** 2)), "first": c2l(u[:4]),
            "last": c2l(u[-4:])}


def main():
    R = RefLib()
    O = Oracle()  # only for the BASELINE shift formula (restated; the reference has no such scheme)
    out = {"generator": "tests/golden/make_golden.py via oracle/_ref (reference grid.cpp/smoother.cpp)"}
    out["rng"] = {str(s): c2l(R.random_complex(s, 12)) for s in (0, 1, 2, 123)}

    # operators on small grids (reference layout, (m, m))
    ops = []
    for n, lam in ((8, 2 - 3j), (10, 100 + 100j), (16, 0.0)):
        m = n - 1
        u = R.random_complex(21, m * m).reshape(m, m)
        b = R.random_complex(22, m * m).reshape(m, m)
        c = R.random_complex(23, (n // 2 - 1) ** 2).reshape(n // 2 - 1, n // 2 - 1)
        ops.append({
            "n": n, "lambda": c2l([lam])[0], "u_seed": 21, "b_seed": 22, "c_seed": 23,
            "vanka": c2l(R.smooth(n, lam, u, b, "vanka", 24 / 25)),
            "jacobi": c2l(R.smooth(n, lam, u, b, "jacobi", 4 / 5)),
            "residual": c2l(R.residual(n, lam, b, u)),
            "restrict": c2l(R.restrict(n, u)),
            "prolong": c2l(R.prolong(n // 2, c)),
        })
    out["operators"] = ops
    out["vanka_coeffs"] = [{"eta": c2l([e])[0], "abc": c2l(R.vanka_coeffs(e))}
                           for e in (0.0, 0.1, 1 + 1j, -0.5j, -1 + 3j)]

    solves = {}
    # BASELINE config 1
    lam = O.circulant_shifts(0.01, 32, 1 / 32, 3, 1)
    b = R.random_complex(0, 63 * 63).reshape(63, 63)
    s = R.solve(64, lam[0], Cfg(), b)
    solves["C1"] = {"n": 64, "lambda": c2l(lam)[0], "seed": 0, "cfg": Cfg().__dict__, "iterations": s["iterations"],
                    "hist": s["hist"].tolist(), "rate": s["rate"], "u": summary(s["u"])}
    # BASELINE config 2: 32 shifts, seed 1 drawn shift-major
    lams = O.circulant_shifts(0.01, 32, 1 / 32)
    b = R.random_complex(1, 32 * 127 * 127).reshape(32, 127, 127)
    s = R.solve_batch(128, lams, Cfg(), b, threads=8)
    solves["C2"] = {"n": 128, "lambdas": c2l(lams), "seed": 1, "cfg": Cfg().__dict__,
                    "iterations": s["iterations"].tolist(),
                    "hist": [s["hist"][j, : s["iterations"][j] + 1].tolist() for j in range(32)],
                    "u": [summary(s["u"][j]) for j in range(32)]}
    # BASELINE config 3 sample: shifts 0 and 128 of 256 (h=1/512, V(2,2), alpha=1e-3)
    lam3 = O.circulant_shifts(1e-3, 256, 1 / 256, 0, 256)[[0, 128]]
    b = R.random_complex(2, 2 * 511 * 511).reshape(2, 511, 511)
    cfg3 = Cfg(nu1=2, nu2=2)
    s = R.solve_batch(512, lam3, cfg3, b, threads=2)
    solves["C3_sample"] = {"n": 512, "shift_indices": [0, 128], "lambdas": c2l(lam3), "seed": 2,
                           "cfg": cfg3.__dict__, "iterations": s["iterations"].tolist(),
                           "hist": [s["hist"][j, : s["iterations"][j] + 1].tolist() for j in range(2)]}
    # README rows (proj/README.md:37-41): W(1,0), h=1/64, coarsest 1/8, tol 1e-8, lambda=0, rhs seed 123
    b = R.random_complex(123, 63 * 63).reshape(63, 63)
    for name, cfg in (("W10_vanka", Cfg(cycle="W", nu1=1, nu2=0, coarsest_n=8, tol=1e-8)),
                      ("W10_jacobi", Cfg(cycle="W", nu1=1, nu2=0, coarsest_n=8, tol=1e-8, smoother="jacobi",
                                         omega=0.8))):
        s = R.solve(64, 0.0, cfg, b)
        solves[name] = {"n": 64, "lambda": [0.0, 0.0], "seed": 123, "cfg": cfg.__dict__,
                        "iterations": s["iterations"], "hist": s["hist"].tolist(), "rate": s["rate"]}
    out["solves"] = solves
    with open(os.path.join(HERE, "reference_golden.json"), "w") as f:
        json.dump(out, f, indent=0)
    print("wrote", os.path.join(HERE, "reference_golden.json"))


if __name__ == "__main__":
    main()
