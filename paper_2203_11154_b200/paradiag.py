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


class _ParadiagBase:
    """A GPU ParaDIAG solver object (pdmg_paradiag_*): one device, or the time slices sharded over `devices`
    (the reference's `threads` argument of paradiag_solve, paradiag.cpp:207-236), with the time transforms
    gathering / scattering across the shards through NVLink peer pointers inside the transform kernels."""

    nt: int
    cfg: MultigridConfig

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

    def parts(self) -> list[tuple[int, int, int]]:
        """Time-slice shards: (first slice, slice count, device)."""
        out = []
        for p in range(N.lib().pdmg_paradiag_num_parts(self._h)):
            t0, cnt, dev = C.c_int32(), C.c_int32(), C.c_int32()
            _check(N.lib().pdmg_paradiag_part_range(self._h, p, C.byref(t0), C.byref(cnt), C.byref(dev)))
            out.append((t0.value, cnt.value, dev.value))
        return out

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

    def run_shards(self, d_f, d_u, want_reports: bool = False):
        """Device-resident run of a sharded solver: d_f[p], d_u[p] = shard p's slices on its device."""
        P_ = len(d_f)
        af, au = (C.c_void_p * P_)(*d_f), (C.c_void_p * P_)(*d_u)
        rr = C.c_double()
        if want_reports:
            rep, it, cv, hist, rate = self._reports()
            _check(N.lib().pdmg_paradiag_run_shards(self._h, af, au, C.byref(rep), C.byref(rr)))
            reps = [SolveReport(bool(cv[s]), int(it[s]), hist[s, : it[s] + 1].copy(), float(rate[s]), rep.seconds)
                    for s in range(self.nt)]
            return reps, rr.value
        _check(N.lib().pdmg_paradiag_run_shards(self._h, af, au, None, C.byref(rr)))
        return None, rr.value


class ParadiagCirculant(_ParadiagBase):
    """GPU ParaDIAG for the alpha-circulant time matrix (alpha > 0: the BASELINE preconditioner; alpha = -1/beta: the
    reference's BackwardHeatQBV)."""

    def __init__(self, grid: Grid2D | int, nt: int, alpha: float, dt: float, cfg: MultigridConfig, device: int = 0,
                 devices=None):
        self.grid = grid if isinstance(grid, Grid2D) else Grid2D(int(grid))
        self.nt, self.alpha, self.dt, self.cfg, self.device = nt, alpha, dt, cfg, device
        self._devs = np.ascontiguousarray(list(devices) if devices else [device], np.int32)
        h = C.c_void_p()
        c = cfg._c()
        _check(N.lib().pdmg_paradiag_create_multi(self.grid.n, nt, alpha, dt, C.byref(c), self._devs.ctypes.data,
                                                  len(self._devs), C.byref(h)))
        self._h = h


class ParadiagGeneral(_ParadiagBase):
    """GPU ParaDIAG for a general diagonalizable time matrix B = V diag(lambdas) V^{-1} (HeatBVM,
    diagonalize_time_matrix, paradiag.cpp:71-82); the time transforms are hand-written complex GEMM kernels."""

    def __init__(self, grid: Grid2D | int, B: np.ndarray, dg: "TimeDiagonalization", cfg: MultigridConfig,
                 device: int = 0, devices=None):
        self.grid = grid if isinstance(grid, Grid2D) else Grid2D(int(grid))
        self.nt, self.cfg, self.device = B.shape[0], cfg, device
        self._B = np.ascontiguousarray(B, np.float64)
        self._lam = np.ascontiguousarray(dg.eigenvalues, np.complex128)
        self._V, self._Vi = np.ascontiguousarray(dg.V, np.complex128), np.ascontiguousarray(dg.Vinv, np.complex128)
        self._devs = np.ascontiguousarray(list(devices) if devices else [device], np.int32)
        h = C.c_void_p()
        c = cfg._c()
        _check(N.lib().pdmg_paradiag_create_general(self.grid.n, self.nt, self._lam.ctypes.data, self._V.ctypes.data,
                                                    self._Vi.ctypes.data, self._B.ctypes.data, C.byref(c),
                                                    self._devs.ctypes.data, len(self._devs), C.byref(h)))
        self._h = h


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


# ---------------------------------------------------------------------------------------------------
# Reference-facing time discretizations (proj/include/pdmg/paradiag.hpp:13-33)
# ---------------------------------------------------------------------------------------------------
import enum as _enum  # noqa: E402
from dataclasses import dataclass as _dataclass  # noqa: E402


class TimeSchemeKind(_enum.IntEnum):
    HeatBVM = 0          # boundary-value-method stencil (general dense eigendecomposition, GEMM time transforms)
    BackwardHeatQBV = 1  # quasi-boundary-value regularization: alpha-circulant with alpha = -1/beta
    CirculantAlpha = 2   # BASELINE's alpha-circulant backward-Euler preconditioner, alpha > 0


@_dataclass(frozen=True)
class TimeDiscretization:
    """pdmg::TimeDiscretization (paradiag.hpp:18-33); `alpha` is used by CirculantAlpha only."""

    kind: TimeSchemeKind = TimeSchemeKind.BackwardHeatQBV
    n: int = 0
    tau: float = 0.0
    beta: float = 0.01
    alpha: float = 0.01

    def dim(self) -> int:  # paradiag.hpp:25
        return self.n + 1 if self.kind == TimeSchemeKind.BackwardHeatQBV else self.n

    def validate(self) -> None:  # paradiag.hpp:27-32
        if self.n < 2:
            raise ConfigError("TimeDiscretization: need n >= 2 time steps")
        if not self.tau > 0.0:
            raise ConfigError("TimeDiscretization: tau must be positive")
        if self.kind == TimeSchemeKind.BackwardHeatQBV and not self.beta > 0.0:
            raise ConfigError("TimeDiscretization: beta must be positive")

    def circulant_alpha(self) -> float:
        if self.kind == TimeSchemeKind.BackwardHeatQBV:
            return -1.0 / self.beta  # paradiag.cpp:209
        if self.kind == TimeSchemeKind.CirculantAlpha:
            return self.alpha
        raise ConfigError("HeatBVM is not circulant: use diagonalize_time_matrix (paradiag.cpp:71-82)")


def time_stepping_matrix(td: TimeDiscretization) -> np.ndarray:
    """Dense B (paradiag.cpp:46-69 for HeatBVM/QBV; C_alpha for CirculantAlpha) -- host-side, for oracles."""
    td.validate()
    it = 1.0 / td.tau
    if td.kind == TimeSchemeKind.HeatBVM:
        n = td.n
        B = np.zeros((n, n))
        for i in range(n - 1):
            B[i, i + 1] = 0.5 * it
            if i > 0:
                B[i, i - 1] = -0.5 * it
        B[n - 1, n - 2] = -it
        B[n - 1, n - 1] = it
        return B
    m = td.dim()
    B = np.zeros((m, m))
    for i in range(m):
        B[i, i] = it
        if i > 0:
            B[i, i - 1] = -it
    B[0, m - 1] = -td.circulant_alpha() * it
    return B


@_dataclass
class TimeDiagonalization:
    """pdmg::TimeDiagonalization (paradiag.hpp:45-53): B = V diag(eigenvalues) V^{-1}."""

    eigenvalues: np.ndarray
    V: np.ndarray
    Vinv: np.ndarray
    cond_estimate: float
    ill_conditioned: bool


def diagonalize_time_matrix(B: np.ndarray) -> TimeDiagonalization:
    """diagonalize_time_matrix (paradiag.cpp:71-82): general dense eigendecomposition (host, setup time; the
    reference uses Eigen::EigenSolver, here LAPACK through numpy).  The eigenvalue order may differ from
    Eigen's; the solution of the space-time system does not depend on it."""
    if B.ndim != 2 or B.shape[0] != B.shape[1] or B.shape[0] < 1:
        raise ConfigError("diagonalize_time_matrix: matrix must be square and nonempty")
    lam, V = np.linalg.eig(B)
    V = V.astype(np.complex128)
    cond = float(np.linalg.cond(V, 1))
    return TimeDiagonalization(lam.astype(np.complex128), V, np.linalg.inv(V), cond, not cond <= 1e12)


def diagonalize_qbv_closed_form(td: TimeDiscretization) -> TimeDiagonalization:
    """diagonalize_qbv_closed_form (paradiag.cpp:84-108): eigenvalue k = (1 - gamma zeta^{-k}) / tau with
    gamma = |alpha|^{1/m} e^{i pi/m}, alpha = -1/beta, zeta = e^{2 pi i/m}; column k of V is
    V(j, k) = gamma^{-j} zeta^{jk} / m, normalized.  cond_estimate is the 1-norm condition number of V (the
    reference's Eigen rcond() estimates the same quantity)."""
    td.validate()
    if td.kind != TimeSchemeKind.BackwardHeatQBV:
        raise ConfigError("diagonalize_qbv_closed_form: scheme is not BackwardHeatQBV")
    m = td.n + 1
    gr, ga, wa = (1.0 / td.beta) ** (1.0 / m), np.pi / m, 2.0 * np.pi / m
    k = np.arange(m)
    lam = (1.0 - gr * np.exp(1j * (ga - wa * k))) / td.tau
    j = np.arange(m)[:, None]
    V = (gr ** (-j.astype(np.float64))) * np.exp(1j * j * (wa * k[None, :] - ga)) / m
    V = V / np.linalg.norm(V, axis=0, keepdims=True)
    cond = float(np.linalg.cond(V, 1))
    return TimeDiagonalization(lam.astype(np.complex128), V, np.linalg.inv(V), cond, not cond <= 1e12)


def qbv_slot_of_reference_index(m: int) -> np.ndarray:
    """The circulant engine's slot q holds lambda_q = (1 - gamma e^{+2 pi i q/m})/tau; the reference's eigenvalue
    k is (1 - gamma zeta^{-k})/tau (paradiag.cpp:100), so reference index k is slot (m - k) mod m."""
    return (m - np.arange(m)) % m


def paradiag_solve(f: np.ndarray, td: TimeDiscretization, cfg: MultigridConfig, device: int = 0, devices=None):
    """paradiag_solve (paradiag.cpp:185-248): returns (u, reports, relres).  The circulant schemes
    (BackwardHeatQBV, CirculantAlpha) transform time with an alpha-scaled FFT; HeatBVM with dense GEMM kernels
    against the eigenvector matrix.  devices: shard the time slices over these devices (the reference's `threads`)."""
    td.validate()
    f = np.ascontiguousarray(f, np.complex128)
    if f.shape[0] != td.dim():
        raise ConfigError(f"paradiag_solve: expected {td.dim()} time slices, got {f.shape[0]}")
    n = f.shape[-1] + 1
    if td.kind != TimeSchemeKind.HeatBVM:
        with ParadiagCirculant(n, td.dim(), td.circulant_alpha(), td.tau, cfg, device, devices) as pd:
            u, reps, rr = pd.run(f)
        if td.kind == TimeSchemeKind.BackwardHeatQBV:  # reports in the reference's eigenvalue order
            reps = [reps[q] for q in qbv_slot_of_reference_index(td.dim())]
        return u, reps, rr
    B = np.ascontiguousarray(time_stepping_matrix(td), np.float64)
    dg = diagonalize_time_matrix(B)
    with ParadiagGeneral(n, B, dg, cfg, device, devices) as pd:
        return pd.run(f)


def helmholtz_shifts(h: float) -> np.ndarray:
    """lambda_j = -j^2 (1 - 0.5 i), j = 1..min(128, floor(1/(2h))) (paradiag.cpp:237-247)."""
    if not (0.0 < h < 0.5):
        raise ConfigError("helmholtz_shifts: need 0 < h < 1/2")
    jmax = min(128, int(np.floor(1.0 / (2.0 * h))))
    j = np.arange(1, jmax + 1, dtype=np.float64)
    return (-(j * j) + 0.5j * (j * j)).astype(np.complex128)


def manufactured_field(grid: Grid2D | int, slices: int, tau: float) -> np.ndarray:
    """u*(x, y, t_i) = sin(pi x) sin(pi y) (1 + t_i), t_i = (i+1) tau (paradiag.cpp:250-267)."""
    n = grid.n if isinstance(grid, Grid2D) else int(grid)
    h = 1.0 / n
    x = np.arange(1, n) * h
    base = np.outer(np.sin(np.pi * x), np.sin(np.pi * x))
    return np.stack([base * (1.0 + (s + 1) * tau) for s in range(slices)]).astype(np.complex128)


def all_at_once_apply(B: np.ndarray, u: np.ndarray) -> np.ndarray:
    """(B (x) I + I (x) A) u, matrix-free over numpy slices (paradiag.cpp:141-161); host-side helper."""
    n = u.shape[-1] + 1
    h2 = 1.0 / n ** 2
    out = np.empty_like(u)
    for i in range(u.shape[0]):
        z = np.pad(u[i], 1)
        au = (4 * z[1:-1, 1:-1] - z[:-2, 1:-1] - z[2:, 1:-1] - z[1:-1, :-2] - z[1:-1, 2:]) / h2
        y = au
        for j in range(u.shape[0]):
            if B[i, j] != 0.0:
                y = y + B[i, j] * u[j]
        out[i] = y
    return out
