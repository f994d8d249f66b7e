"""ParaDIAG with the alpha-circulant backward-Euler time matrix on the GPU (reference driver:
proj/src/paradiag.cpp:185-248; its time transforms kron_time_solve/kron_time_apply, paradiag.cpp:129-139,
become an alpha-scaled DFT over the time index, and step 2 is the batched multigrid solve).

    C_alpha = (1/dt)(I - Sigma_alpha),  Sigma_alpha = down-shift with corner alpha at (0, nt-1)
    step 1  g = ifft_t(alpha^(t/nt) f)
    step 2  (A + lambda_k I) w_k = g_k,   lambda_k = (1 - alpha^(1/nt) e^(2 pi i k/nt)) / dt
    step 3  u = alpha^(-t/nt) fft_k(w)
    relres  = ||f - (C_alpha (x) I + I (x) A) u|| / ||f||      (paradiag.cpp:243-245)

Arrays are [nt][m][m] complex128 time slices (reference layout).  Multi-GPU: `paradiag_distributed`
shards time slices over ranks and moves data with NCCL all-to-all around the time DFT.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .multigrid import ConfigError, Grid2D, MultigridConfig, SolveReport, _check


class ParadiagCirculant:
    """GPU ParaDIAG solver for one (n, nt, alpha, dt, cfg) on one device."""

    def __init__(self, grid: Grid2D | int, nt: int, alpha: float, dt: float, cfg: MultigridConfig, device: int = 0):
        self.grid = grid if isinstance(grid, Grid2D) else Grid2D(int(grid))
        self.nt, self.alpha, self.dt, self.cfg, self.device = nt, alpha, dt, cfg, device
        h = C.c_void_p()
        c = cfg._c()
        _check(N.lib().pdmg_paradiag_create(self.grid.n, nt, alpha, dt, C.byref(c), device, C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            N.lib().pdmg_paradiag_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *e):
        self.close()

    @property
    def solver_handle(self):
        return N.lib().pdmg_paradiag_solver(self._h)

    def _reports(self):
        S, H = self.nt, self.cfg.max_iter + 1
        it = np.zeros(S, np.int32)
        cv = np.zeros(S, np.uint8)
        hist = np.zeros((S, H), np.float64)
        rate = np.zeros(S, np.float64)
        return N.SolveReport(it.ctypes.data, cv.ctypes.data, hist.ctypes.data, rate.ctypes.data, 0.0), it, cv, hist, rate

    def run(self, f: np.ndarray):
        m = self.grid.n - 1
        ff = np.ascontiguousarray(f, np.complex128)
        if ff.shape != (self.nt, m, m):
            raise ConfigError(f"paradiag_solve: expected {(self.nt, m, m)} time slices, got {ff.shape}")
        u = np.empty_like(ff)
        rep, it, cv, hist, rate = self._reports()
        rr = C.c_double()
        _check(N.lib().pdmg_paradiag_run(self._h, ff.ctypes.data, u.ctypes.data, C.byref(rep), C.byref(rr)))
        reps = [SolveReport(bool(cv[s]), int(it[s]), hist[s, : it[s] + 1].copy(), float(rate[s]), rep.seconds)
                for s in range(self.nt)]
        return u, reps, rr.value

    def run_device(self, d_f: int, d_u: int):
        rr = C.c_double()
        _check(N.lib().pdmg_paradiag_run_device(self._h, d_f, d_u, None, C.byref(rr)))
        return rr.value


def heat_initial_rhs(n: int, nt: int, dt: float, seed: int = 4) -> np.ndarray:
    """BASELINE config 5 right-hand side: u0 = sin(pi x) sin(pi y) + uniform[-0.1, 0.1] (std::mt19937(seed),
    one real draw per node, x fastest), all-at-once backward Euler f_1 = u0/dt, f_{t>1} = 0."""
    m = n - 1
    h = 1.0 / n
    x = np.arange(1, n) * h
    u0 = np.outer(np.sin(np.pi * x), np.sin(np.pi * x))
    # the perturbation uses the same engine/distribution as the reference RHS generator (pdmg.cpp:137-147)
    draws = _real_draws(seed, -0.1, 0.1, m * m)
    f = np.zeros((nt, m, m), np.complex128)
    f[0] = (u0 + draws.reshape(m, m)) / dt
    return f


def _real_draws(seed: int, lo: float, hi: float, count: int) -> np.ndarray:
    """One real uniform draw per node from std::mt19937(seed): the complex generator draws (re, im) pairs
    from the same stream, so reading its output as a flat real array gives the real sequence."""
    buf = np.empty((count + 1) // 2, np.complex128)
    N.lib().pdmg_random_rhs(seed, lo, hi, buf.size, buf.ctypes.data)
    return buf.view(np.float64)[:count].copy()
