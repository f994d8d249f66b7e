"""numpy restatement of the reference's local Fourier analysis (proj/src/lfa.cpp:68-248) -- TEST INFRASTRUCTURE ONLY.

The two-grid spectral radius uses numpy's LAPACK eigenvalue solver on the same 4 x 4 matrices the reference hands to
Eigen::ComplexEigenSolver (lfa.cpp:39-45).  Pinned in tests/test_lfa.py against the reference's own published values
(proj/README.md:108-112) and known answers (proj/tests/test_lfa.cpp, acceptance.cpp:82-139).
"""
from __future__ import annotations

import math

import numpy as np

PI = math.pi
TIE = 1e-12  # lfa.cpp:15


def vanka_coeffs(eta: complex):  # smoother.cpp:18-29
    i2, i4, i6 = 1 / (2 + eta), 1 / (4 + eta), 1 / (6 + eta)
    return 0.25 * (i2 + 2 * i4 + i6), 0.25 * (i2 - i6), 0.25 * (i2 - 2 * i4 + i6)


def sym_L(t1, t2, lam, h):  # lfa.cpp:68-71
    return (4.0 - 2.0 * np.cos(t1) - 2.0 * np.cos(t2) + lam * h * h) / (h * h)


def sym_M(t1, t2, lam, h, kind):  # lfa.cpp:73-82
    eta = lam * h * h
    if kind == "jacobi":
        return np.full(np.shape(t1), h * h / (4 + eta), np.complex128)
    a, b, c = vanka_coeffs(eta)
    c1, c2 = np.cos(t1), np.cos(t2)
    return (h * h) * (a + b * (c1 + c2) + c * (c1 * c2))


def sym_R(t1, t2):  # lfa.cpp:89-91
    return 0.25 * (1 + np.cos(t1)) * (1 + np.cos(t2))


def base_thetas(n):
    return -0.5 * PI + np.arange(n) * (PI / n)


def high_frequencies(n):
    """theta1 outer, theta2 inner, shifts (1,0), (0,1), (1,1) innermost (lfa.cpp:31-37)."""
    th = base_thetas(n)
    t1 = np.repeat(th, n * 3)
    t2 = np.tile(np.repeat(th, 3), n)
    s = np.tile(np.array([[1, 0], [0, 1], [1, 1]]), (n * n, 1))
    return t1 + PI * s[:, 0], t2 + PI * s[:, 1]


def first_max(v, t1, t2):
    best, at = -1.0, 0
    for q, x in enumerate(v):
        if x > best + TIE:
            best, at = x, q
    return best, (t1[at], t2[at])


def smoothing_factor(lam, h, kind, omega, n=64):
    t1, t2 = high_frequencies(n)
    v = np.abs(1 - omega * sym_M(t1, t2, lam, h, kind) * sym_L(t1, t2, lam, h))
    return first_max(v, t1, t2)


def smoothing_factor_bound(lam, h, omega, n=64):
    t1, t2 = high_frequencies(n)
    base = np.abs(1 - omega * sym_M(t1, t2, 0.0, h, "vanka") * sym_L(t1, t2, 0.0, h)).max()
    shift = np.abs(omega * lam * sym_M(t1, t2, lam, h, "vanka")).max()
    return base, shift


class TwoGridModel:
    """lfa.cpp:117-174."""

    def __init__(self, lam, h, kind, n=64, skip_tol=1e-8):
        th = base_thetas(n)
        T1, T2 = np.meshgrid(th, th, indexing="ij")
        t1, t2 = T1.ravel(), T2.ravel()
        h1 = np.stack([t1, t1 + PI, t1, t1 + PI], 1)
        h2 = np.stack([t2, t2, t2 + PI, t2 + PI], 1)
        L = sym_L(h1, h2, lam, h)
        ML = sym_M(h1, h2, lam, h, kind) * L
        R = sym_R(h1, h2)
        Lc = sym_L(2 * t1, 2 * t2, lam, 2 * h)
        keep = np.abs(Lc) > skip_tol
        self.skipped = int(np.sum(~keep))
        self.ml = ML[keep]
        Rk, Lk, Lck = R[keep], L[keep], Lc[keep]
        self.cgc = np.eye(4)[None] - Rk[:, :, None] * Rk[:, None, :] * Lk[:, None, :] / Lck[:, None, None]
        self.high_ml = ML[:, 1:].ravel()
        self.high_t1, self.high_t2 = h1[:, 1:].ravel(), h2[:, 1:].ravel()

    def rho(self, omega, nu):
        s = (1 - omega * self.ml) ** nu
        E = s[:, :, None] * self.cgc
        return float(np.abs(np.linalg.eigvals(E)).max())

    def smoothing(self, omega):
        return first_max(np.abs(1 - omega * self.high_ml), self.high_t1, self.high_t2)


def minimize_scalar(f):  # lfa.cpp:183-219
    lo, hi, step = 0.1, 1.9, 0.01
    nsteps = int(round((hi - lo) / step))
    best_w, best_v = lo, f(lo)
    for k in range(1, nsteps + 1):
        w = lo + k * step
        v = f(w)
        if v < best_v:
            best_w, best_v = w, v
    a, b = max(lo, best_w - step), min(hi, best_w + step)
    invphi = (math.sqrt(5.0) - 1.0) / 2.0
    x1, x2 = b - invphi * (b - a), a + invphi * (b - a)
    f1, f2 = f(x1), f(x2)
    while b - a > 1e-4:
        if f1 <= f2:
            b, x2, f2 = x2, x1, f1
            x1 = b - invphi * (b - a)
            f1 = f(x1)
        else:
            a, x1, f1 = x1, x2, f2
            x2 = a + invphi * (b - a)
            f2 = f(x2)
    w = 0.5 * (a + b)
    return w, f(w)
