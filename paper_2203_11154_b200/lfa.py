"""Local Fourier analysis on the GPU (mirror of proj/include/pdmg/lfa.hpp over the C ABI; restating proj/src/lfa.cpp).

Names follow the reference: `FrequencyPair`, `LFAConfig`, `symbol_shifted_laplacian`, `symbol_vanka`,
`symbol_preconditioner`, `symbol_smoother_error`, `symbol_transfer`, `SmoothingReport`, `smoothing_factor`,
`SmoothingBound`, `smoothing_factor_bound`, `TwoGridModel` (rho, smoothing, skipped_bases), `two_grid_factor`,
`OmegaObjective`, `OmegaOpt`, `optimize_omega`.  The per-frequency work (symbols on the sampled grid, the 4 x 4
two-grid spectral radii for every base and damping) runs in libpdmg_b200.so's LFA kernels.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass

from . import _native as N
from .multigrid import ConfigError, Shift, SmootherConfig, SmootherKind, _check


@dataclass(frozen=True)
class FrequencyPair:
    t1: float = 0.0
    t2: float = 0.0


@dataclass(frozen=True)
class LFAConfig:
    """lfa.hpp:21-31."""

    samples_per_dim: int = 64
    coarse_skip_tol: float = 1e-8

    def validate(self) -> None:
        if self.samples_per_dim < 16 or self.samples_per_dim % 2 != 0:
            raise ConfigError("LFAConfig: samples_per_dim must be even and >= 16")
        if not self.coarse_skip_tol > 0.0:
            raise ConfigError("LFAConfig: coarse_skip_tol must be positive")

    def _c(self):
        return N.LfaConfig(self.samples_per_dim, self.coarse_skip_tol)


def _shift(s) -> N.C128:
    lam = complex(s.lam if isinstance(s, Shift) else s)
    return N.C128(lam.real, lam.imag)


def _symbol(which: int, th: FrequencyPair, shift, h: float, kind: int = 0, omega: float = 0.0) -> complex:
    out = N.C128()
    _check(N.lib().pdmg_lfa_symbol(which, th.t1, th.t2, _shift(shift), h, int(kind), omega, C.byref(out)))
    return complex(out.re, out.im)


def symbol_shifted_laplacian(th: FrequencyPair, shift, h: float) -> complex:
    return _symbol(0, th, shift, h)


def symbol_vanka(th: FrequencyPair, shift, h: float) -> complex:
    return _symbol(1, th, shift, h)


def symbol_preconditioner(th: FrequencyPair, shift, h: float, kind: SmootherKind) -> complex:
    return _symbol(2, th, shift, h, kind)


def symbol_smoother_error(th: FrequencyPair, shift, h: float, cfg: SmootherConfig) -> complex:
    return _symbol(3, th, shift, h, cfg.kind, cfg.omega)


def symbol_transfer(th: FrequencyPair) -> float:
    return _symbol(4, th, 0.0, 1.0).real


@dataclass
class SmoothingReport:
    mu: float = 0.0
    argmax: FrequencyPair = FrequencyPair()


@dataclass
class SmoothingBound:
    phi_base: float = 0.0
    phi_shift: float = 0.0

    def total(self) -> float:
        return self.phi_base + self.phi_shift


def smoothing_factor(shift, h: float, cfg: SmootherConfig, lfa: LFAConfig = LFAConfig(), device: int = 0):
    mu, arg = C.c_double(), (C.c_double * 2)()
    c = lfa._c()
    _check(N.lib().pdmg_lfa_smoothing_factor(_shift(shift), h, int(cfg.kind), cfg.omega, C.byref(c), device,
                                             C.byref(mu), arg))
    return SmoothingReport(mu.value, FrequencyPair(arg[0], arg[1]))


def smoothing_factor_bound(shift, h: float, omega: float, lfa: LFAConfig = LFAConfig(), device: int = 0):
    phi = (C.c_double * 2)()
    c = lfa._c()
    _check(N.lib().pdmg_lfa_smoothing_bound(_shift(shift), h, omega, C.byref(c), device, phi))
    return SmoothingBound(phi[0], phi[1])


class OmegaObjective(enum.IntEnum):
    TwoGridRho = 0
    SmoothingMu = 1


@dataclass
class OmegaOpt:
    omega: float = 0.0
    value: float = 0.0


class TwoGridModel:
    """lfa.hpp:77-96: two-grid error model with its symbol caches on the device."""

    def __init__(self, shift, h: float, kind: SmootherKind, lfa: LFAConfig = LFAConfig(), device: int = 0):
        h_ = C.c_void_p()
        c = lfa._c()
        _check(N.lib().pdmg_lfa_model_create(_shift(shift), h, int(kind), C.byref(c), device, C.byref(h_)))
        self._h = h_

    def close(self):
        if getattr(self, "_h", None):
            N.lib().pdmg_lfa_model_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def rho(self, omega, nu: int):
        """rho(omega, nu); omega may be a sequence (one GPU launch for the whole batch)."""
        ws = [float(omega)] if isinstance(omega, (int, float)) else [float(w) for w in omega]
        arr, out = (C.c_double * len(ws))(*ws), (C.c_double * len(ws))()
        _check(N.lib().pdmg_lfa_model_rho(self._h, len(ws), arr, nu, out))
        return out[0] if isinstance(omega, (int, float)) else list(out)

    def smoothing(self, omega: float) -> SmoothingReport:
        mu, arg = C.c_double(), (C.c_double * 2)()
        _check(N.lib().pdmg_lfa_model_smoothing(self._h, omega, C.byref(mu), arg))
        return SmoothingReport(mu.value, FrequencyPair(arg[0], arg[1]))

    def skipped_bases(self) -> int:
        return N.lib().pdmg_lfa_model_skipped(self._h)


def two_grid_factor(shift, h: float, cfg: SmootherConfig, nu: int, lfa: LFAConfig = LFAConfig(), device: int = 0):
    return TwoGridModel(shift, h, cfg.kind, lfa, device).rho(cfg.omega, nu)


def optimize_omega(model_or_shift, *args, **kw) -> OmegaOpt:
    """optimize_omega(model, objective, nu=1) or optimize_omega(shift, h, kind, objective, nu=1, lfa=LFAConfig())
    (lfa.hpp:105-117)."""
    w, v = C.c_double(), C.c_double()
    if isinstance(model_or_shift, TwoGridModel):
        objective = args[0] if args else kw["objective"]
        nu = args[1] if len(args) > 1 else kw.get("nu", 1)
        _check(N.lib().pdmg_lfa_optimize_omega(model_or_shift._h, int(objective), nu, C.byref(w), C.byref(v)))
        return OmegaOpt(w.value, v.value)
    h, kind, objective = args[0], args[1], args[2]
    nu = args[3] if len(args) > 3 else kw.get("nu", 1)
    lfa = args[4] if len(args) > 4 else kw.get("lfa", LFAConfig())
    device = kw.get("device", 0)
    if OmegaObjective(objective) == OmegaObjective.TwoGridRho:
        return optimize_omega(TwoGridModel(model_or_shift, h, kind, lfa, device), objective, nu)
    c = lfa._c()
    _check(N.lib().pdmg_lfa_optimize_omega_smoothing(_shift(model_or_shift), h, int(kind), C.byref(c), device,
                                                     C.byref(w), C.byref(v)))
    return OmegaOpt(w.value, v.value)
