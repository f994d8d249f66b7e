"""Host-side mirror of the reference `pdmg::` solver interface over the B200 C ABI.

Names, argument meaning and error behaviour follow the reference (He & Liu, arXiv 2203.11154, artifact
`pdmg`): `Grid2D`, `Shift` (proj/include/pdmg/grid.hpp:16-52), `SmootherConfig`
(proj/include/pdmg/smoother.hpp:30-38), `MultigridConfig`, `SolveReport`, `MultigridHierarchy`,
`multigrid_solve` (proj/include/pdmg/multigrid.hpp:12-83), `ConfigError` / `SingularOperatorError`
(proj/include/pdmg/errors.hpp:10-28).  The one deliberate extension is batching:
`BatchedMultigridHierarchy` holds one hierarchy per shift and advances all of them together on the GPU,
which is what `paradiag_solve`'s loop over shifts (proj/src/paradiag.cpp:207-236) becomes.

Grid functions are numpy complex128 arrays in the reference layout: interior nodes only, shape
(m, m) = (n-1, n-1) with x fastest (array[j-1, i-1] is node (i, j)); batches are (n_shifts, m, m).
Every computation runs in libpdmg_b200.so on the GPU -- there is no CPU path here.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Iterable, Sequence

import numpy as np

from . import _native as N


class ConfigError(ValueError):
    """pdmg::ConfigError (errors.hpp:12-15): invalid sizes or configuration."""


class SingularOperatorError(RuntimeError):
    """pdmg::SingularOperatorError (errors.hpp:20-23): a required operator is singular."""


class DeviceError(RuntimeError):
    """CUDA / device failure (status 3)."""


def _check(status: int) -> None:
    if status == N.PDMG_OK:
        return
    msg = N.lib().pdmg_last_error().decode()
    if status == N.PDMG_ERR_CONFIG:
        raise ConfigError(msg)
    if status == N.PDMG_ERR_SINGULAR:
        raise SingularOperatorError(msg)
    raise DeviceError(msg)


class CycleKind(enum.IntEnum):
    V = 0
    W = 1


class SmootherKind(enum.IntEnum):
    Vanka = 0
    Jacobi = 1


@dataclass(frozen=True)
class Grid2D:
    """Uniform vertex-centred grid on the unit square, h = 1/n, (n-1)^2 interior nodes (grid.hpp:16-36)."""

    n: int

    def __post_init__(self):
        if self.n < 2:
            raise ConfigError(f"Grid2D: need at least 2 subdivisions per side, got {self.n}")

    @property
    def h(self) -> float:
        return 1.0 / self.n

    def interior_per_side(self) -> int:
        return self.n - 1

    def size(self) -> int:
        return (self.n - 1) ** 2

    def coarsenable(self) -> bool:
        return self.n % 2 == 0 and self.n >= 4

    def coarse(self) -> "Grid2D":
        if not self.coarsenable():
            raise ConfigError(f"Grid2D: cannot coarsen grid with n = {self.n}")
        return Grid2D(self.n // 2)


class ShiftKind(enum.IntEnum):
    User = 0
    TimeEigenvalue = 1
    Helmholtz = 2


@dataclass(frozen=True)
class Shift:
    """Complex shift lambda of A + lambda I (grid.hpp:44-52)."""

    lam: complex = 0j
    index: int = 0
    kind: ShiftKind = ShiftKind.User

    def eta(self, h: float) -> complex:
        return complex(self.lam) * (h * h)


@dataclass(frozen=True)
class SmootherConfig:
    kind: SmootherKind = SmootherKind.Vanka
    omega: float = 24.0 / 25.0

    @staticmethod
    def vanka(w: float = 24.0 / 25.0) -> "SmootherConfig":
        return SmootherConfig(SmootherKind.Vanka, w)

    @staticmethod
    def jacobi(w: float = 4.0 / 5.0) -> "SmootherConfig":
        return SmootherConfig(SmootherKind.Jacobi, w)


@dataclass(frozen=True)
class MultigridConfig:
    """Defaults are the reference's: W(1,0), coarsest_n 8, tol 1e-8, max_iter 200 (multigrid.hpp:14-23)."""

    cycle: CycleKind = CycleKind.W
    nu1: int = 1
    nu2: int = 0
    coarsest_n: int = 8
    tol: float = 1e-8
    max_iter: int = 200
    smoother: SmootherConfig = field(default_factory=SmootherConfig)

    def validate(self) -> None:  # multigrid.hpp:25-31
        if self.nu1 < 0 or self.nu2 < 0:
            raise ConfigError("MultigridConfig: negative smoothing counts")
        if self.nu1 + self.nu2 == 0:
            raise ConfigError("MultigridConfig: nu1 + nu2 must be positive")
        if self.coarsest_n < 2:
            raise ConfigError("MultigridConfig: coarsest_n must be >= 2")
        if not self.tol > 0.0:
            raise ConfigError("MultigridConfig: tol must be positive")
        if self.max_iter < 1:
            raise ConfigError("MultigridConfig: max_iter must be >= 1")

    def _c(self) -> N.MgConfig:
        return N.MgConfig(int(self.cycle), self.nu1, self.nu2, self.coarsest_n, self.tol, self.max_iter,
                          int(self.smoother.kind), self.smoother.omega)


@dataclass
class SolveReport:
    """pdmg::SolveReport (multigrid.hpp:34-44)."""

    converged: bool = False
    iterations: int = 0
    residual_history: np.ndarray = field(default_factory=lambda: np.zeros(0))
    rate: float = 0.0
    seconds: float = 0.0


def _as_batch(a, S: int, m: int, name: str) -> np.ndarray:
    arr = np.ascontiguousarray(a, dtype=np.complex128)
    if arr.shape == (m, m) and S == 1:
        arr = arr.reshape(1, m, m)
    if arr.shape != (S, m, m):
        raise ConfigError(f"{name}: expected shape {(S, m, m)}, got {arr.shape} (grid mismatch)")
    return arr


class BatchedMultigridHierarchy:
    """One multigrid hierarchy per shift on a shared fine grid, advanced together on one GPU.

    Construction validates exactly what `MultigridHierarchy(Grid2D, Shift, MultigridConfig)` validates
    (multigrid.cpp:24-61) for every shift, before touching the device.
    """

    def __init__(self, fine: Grid2D, shifts: Sequence[Shift | complex], cfg: MultigridConfig, device: int = 0,
                 precision: str = "c128", devices: Sequence[int] | None = None):
        """precision: "c128" (the reference's std::complex<double>) or "c64" (fp32 storage, fp64 arithmetic;
        host arrays stay complex128).  devices: shard the shifts over these devices (contiguous chunks of
        ceil(S / len(devices)), paradiag.cpp:217-236), one engine and host thread per shard."""
        if isinstance(fine, int):
            fine = Grid2D(fine)
        if precision not in ("c128", "c64"):
            raise ConfigError(f"unknown precision {precision!r}")
        self.precision = precision
        self.grid = fine
        self.cfg = cfg
        self.shifts = [s if isinstance(s, Shift) else Shift(complex(s), i) for i, s in enumerate(shifts)]
        self.device = device
        lam = np.array([complex(s.lam) for s in self.shifts], dtype=np.complex128)
        self._lam = lam
        self.devices = list(devices) if devices else None
        self._devs = np.ascontiguousarray(self.devices or [], np.int32)
        desc = N.BatchDesc(fine.n, len(lam), lam.ctypes.data, cfg._c(), 0 if precision == "c128" else 1, device,
                           self._devs.ctypes.data if self.devices else None, len(self._devs))
        h = C.c_void_p()
        _check(N.lib().pdmg_create(C.byref(desc), C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            N.lib().pdmg_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- structure ---------------------------------------------------------------------------
    @property
    def n_shifts(self) -> int:
        return len(self.shifts)

    def num_levels(self) -> int:
        return N.lib().pdmg_num_levels(self._h)

    def level_grid(self, ell: int) -> Grid2D:
        n = N.lib().pdmg_level_n(self._h, ell)
        if n < 0:
            raise ConfigError(f"level index {ell} out of range")
        return Grid2D(n)

    def coarse_singular(self, s: int) -> bool:
        return bool(N.lib().pdmg_coarse_singular(self._h, s))

    @property
    def stream(self) -> int:
        return N.lib().pdmg_stream(self._h)

    # -- solve -------------------------------------------------------------------------------
    def _report_bufs(self):
        S, H = self.n_shifts, self.cfg.max_iter + 1
        it = np.zeros(S, np.int32)
        cv = np.zeros(S, np.uint8)
        hist = np.zeros((S, H), np.float64)
        rate = np.zeros(S, np.float64)
        rep = N.SolveReport(it.ctypes.data, cv.ctypes.data, hist.ctypes.data, rate.ctypes.data, 0.0)
        return rep, it, cv, hist, rate

    @staticmethod
    def _reports(rep, it, cv, hist, rate) -> list[SolveReport]:
        return [SolveReport(bool(cv[s]), int(it[s]), hist[s, : it[s] + 1].copy(), float(rate[s]), rep.seconds)
                for s in range(it.size)]

    def solve(self, b) -> tuple[np.ndarray, list[SolveReport]]:
        """MultigridHierarchy::solve for every shift from u = 0 (multigrid.cpp:85-110)."""
        m = self.grid.n - 1
        bb = _as_batch(b, self.n_shifts, m, "MultigridHierarchy::solve")
        u = np.empty_like(bb)
        rep, it, cv, hist, rate = self._report_bufs()
        _check(N.lib().pdmg_solve(self._h, bb.ctypes.data, u.ctypes.data, C.byref(rep)))
        return u, self._reports(rep, it, cv, hist, rate)

    def solve_device(self, d_b: int, d_u: int, want_reports: bool = True):
        """Solve with b and u already in device memory (compact layout); returns the reports."""
        if want_reports:
            rep, it, cv, hist, rate = self._report_bufs()
            _check(N.lib().pdmg_solve_device(self._h, d_b, d_u, C.byref(rep)))
            return self._reports(rep, it, cv, hist, rate)
        _check(N.lib().pdmg_solve_device(self._h, d_b, d_u, None))
        return None

    def parts(self) -> list[tuple[int, int, int]]:
        """Device shards: (first shift, shift count, device) per shard."""
        out = []
        for p in range(N.lib().pdmg_num_parts(self._h)):
            s0, cnt, dev = C.c_int32(), C.c_int32(), C.c_int32()
            _check(N.lib().pdmg_part_range(self._h, p, C.byref(s0), C.byref(cnt), C.byref(dev)))
            out.append((s0.value, cnt.value, dev.value))
        return out

    def solve_device_shards(self, d_b: Sequence[int], d_u: Sequence[int], want_reports: bool = True):
        """Solve with each shard's b and u already in its device's memory (pdmg_solve_device_shards)."""
        P_ = len(d_b)
        arr_b, arr_u = (C.c_void_p * P_)(*d_b), (C.c_void_p * P_)(*d_u)
        if want_reports:
            rep, it, cv, hist, rate = self._report_bufs()
            _check(N.lib().pdmg_solve_device_shards(self._h, arr_b, arr_u, C.byref(rep)))
            return self._reports(rep, it, cv, hist, rate)
        _check(N.lib().pdmg_solve_device_shards(self._h, arr_b, arr_u, None))
        return None

    def cycle(self, u, b) -> np.ndarray:
        """MultigridHierarchy::cycle applied to every shift; returns the updated u (multigrid.cpp:79-83)."""
        m = self.grid.n - 1
        uu = _as_batch(u, self.n_shifts, m, "MultigridHierarchy::cycle").copy()
        bb = _as_batch(b, self.n_shifts, m, "MultigridHierarchy::cycle")
        _check(N.lib().pdmg_cycle(self._h, uu.ctypes.data, bb.ctypes.data))
        return uu

    # -- level operators (batched over shifts) -----------------------------------------------
    def _m(self, ell: int) -> int:
        return self.level_grid(ell).n - 1

    def apply_smoother(self, ell: int, u, b) -> np.ndarray:
        m = self._m(ell)
        uu, bb = _as_batch(u, self.n_shifts, m, "apply_smoother"), _as_batch(b, self.n_shifts, m, "apply_smoother")
        out = np.empty_like(uu)
        _check(N.lib().pdmg_apply_smoother(self._h, ell, uu.ctypes.data, bb.ctypes.data, out.ctypes.data))
        return out

    def residual(self, ell: int, b, u) -> np.ndarray:
        m = self._m(ell)
        uu, bb = _as_batch(u, self.n_shifts, m, "residual"), _as_batch(b, self.n_shifts, m, "residual")
        out = np.empty_like(uu)
        _check(N.lib().pdmg_residual(self._h, ell, bb.ctypes.data, uu.ctypes.data, out.ctypes.data))
        return out

    def restrict_full_weighting(self, ell: int, fine) -> np.ndarray:
        m = self._m(ell)
        ff = _as_batch(fine, self.n_shifts, m, "restrict_full_weighting")
        mc = self._m(ell + 1)
        out = np.empty((self.n_shifts, mc, mc), np.complex128)
        _check(N.lib().pdmg_restrict_full_weighting(self._h, ell, ff.ctypes.data, out.ctypes.data))
        return out

    def prolong_bilinear(self, ell: int, coarse) -> np.ndarray:
        mc = self._m(ell + 1)
        cc = _as_batch(coarse, self.n_shifts, mc, "prolong_bilinear")
        m = self._m(ell)
        out = np.empty((self.n_shifts, m, m), np.complex128)
        _check(N.lib().pdmg_prolong_bilinear(self._h, ell, cc.ctypes.data, out.ctypes.data))
        return out

    def norm(self, ell: int, v) -> np.ndarray:
        m = self._m(ell)
        vv = _as_batch(v, self.n_shifts, m, "norm")
        out = np.empty(self.n_shifts, np.float64)
        _check(N.lib().pdmg_norm(self._h, ell, vv.ctypes.data, out.ctypes.data))
        return out

    def coarse_solve(self, b) -> np.ndarray:
        ell = self.num_levels() - 1
        m = self._m(ell)
        bb = _as_batch(b, self.n_shifts, m, "DenseShiftedSolver::solve")
        out = np.empty_like(bb)
        _check(N.lib().pdmg_coarse_solve(self._h, bb.ctypes.data, out.ctypes.data))
        return out

    # -- instrumentation ---------------------------------------------------------------------
    def set_solve_path(self, path: str) -> None:
        """'auto', 'batched' (level passes over all shifts) or 'small' (one CTA per shift, one launch)."""
        _check(N.lib().pdmg_set_solve_path(self._h, {"auto": 0, "batched": 1, "small": 2}[path]))

    def set_profiling(self, on: bool) -> None:
        _check(N.lib().pdmg_set_profiling(self._h, 1 if on else 0))

    def reset_stats(self) -> None:
        N.lib().pdmg_reset_stats(self._h)

    def launch_count(self) -> int:
        return int(N.lib().pdmg_launch_count(self._h))

    def last_updates(self) -> float:
        return float(N.lib().pdmg_last_updates(self._h))

    def kernel_stats(self) -> dict[str, dict]:
        return kernel_stats(self._h)


def kernel_stats(handle) -> dict[str, dict]:
    """Per-kernel-class CUDA-event stats of a pdmg_ctx (pdmg_kernel_stats / pdmg_kernel_updates)."""
    out = {}
    i = 0
    name = C.create_string_buffer(128)
    while True:
        la, ms, by = C.c_int64(), C.c_double(), C.c_double()
        if N.lib().pdmg_kernel_stats(handle, i, name, 128, C.byref(la), C.byref(ms), C.byref(by)):
            break
        ub, nu = C.c_double(), C.c_double()
        N.lib().pdmg_kernel_updates(handle, i, C.byref(ub), C.byref(nu))
        out[name.value.decode()] = dict(launches=la.value, ms=ms.value, bytes=by.value, unit_bytes=ub.value,
                                        updates=nu.value)
        i += 1
    return out


class MultigridHierarchy:
    """Single-shift hierarchy with the reference's call shapes (multigrid.hpp:50-78)."""

    def __init__(self, fine: Grid2D, shift: Shift | complex, cfg: MultigridConfig, device: int = 0):
        self._b = BatchedMultigridHierarchy(fine, [shift], cfg, device)
        self.grid = self._b.grid

    def num_levels(self) -> int:
        return self._b.num_levels()

    def level_grid(self, ell: int) -> Grid2D:
        return self._b.level_grid(ell)

    def cycle(self, u: np.ndarray, b: np.ndarray) -> None:
        """In place, like `void cycle(GridFunction& u, const GridFunction& b) const`."""
        u[...] = self._b.cycle(u, b).reshape(u.shape)

    def solve(self, u: np.ndarray, b: np.ndarray) -> SolveReport:
        """Fills u (overwritten from the zero guess) and returns the report."""
        uu, reps = self._b.solve(b)
        u[...] = uu.reshape(u.shape)
        return reps[0]


def multigrid_solve(b: np.ndarray, shift: Shift | complex, cfg: MultigridConfig, device: int = 0):
    """Convenience driver (multigrid.cpp:112-118): returns (u, SolveReport)."""
    m = b.shape[-1]
    h = MultigridHierarchy(Grid2D(m + 1), shift, cfg, device)
    u = np.zeros_like(np.asarray(b, np.complex128))
    rep = h.solve(u, b)
    return u, rep


def random_rhs(grid: Grid2D | int, seed: int, count: int = 1, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    """tools/pdmg.cpp:137-147 (std::mt19937 + uniform_real_distribution, re then im), `count` grid functions
    drawn from one stream, shift-major.  Host-only (no GPU needed)."""
    n = grid.n if isinstance(grid, Grid2D) else int(grid)
    m = n - 1
    out = np.empty((count, m, m), np.complex128)
    N.lib().pdmg_random_rhs(seed, lo, hi, count * m * m, out.ctypes.data)
    return out[0] if count == 1 else out


def circulant_shifts(alpha: float, nt: int, dt: float, j0: int = 0, count: int | None = None) -> np.ndarray:
    """lambda_j = (1 - alpha^(1/nt) e^(2 pi i j / nt)) / dt (BASELINE.json shift family)."""
    count = nt if count is None else count
    out = np.empty(count, np.complex128)
    N.lib().pdmg_circulant_shifts(alpha, nt, dt, j0, count, out.ctypes.data)
    return out
