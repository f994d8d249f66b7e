"""ctypes bindings for the CPU oracle (TEST INFRASTRUCTURE ONLY).

`Oracle` wraps oracle/liboracle.so (the plain-C restatement, travels to the GPU box) and `RefLib`
wraps oracle/_ref/libpdmg_ref.so (the reference's own grid.cpp/smoother.cpp + restated driver; only
built where /root/reference exists).  Only tests/, __graft_entry__.smoke() and bench.py's CPU legs
import this module.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libpdmg_ref.so")

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_cp = np.ctypeslib.ndpointer(dtype=np.complex128, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")


class _Cplx(C.Structure):
    """By-value `double _Complex` (x86-64 SysV passes it like struct {double re, im;} in two SSE regs)."""

    _fields_ = [("re", C.c_double), ("im", C.c_double)]


class OrcConfig(C.Structure):
    """orc_config (oracle/pdmg_oracle.h) == MultigridConfig (proj/include/pdmg/multigrid.hpp:14-32)."""

    _fields_ = [("cycle", C.c_int), ("nu1", C.c_int), ("nu2", C.c_int), ("coarsest_n", C.c_int),
                ("max_iter", C.c_int), ("smoother", C.c_int), ("tol", C.c_double), ("omega", C.c_double)]


@dataclass
class Cfg:
    cycle: str = "V"
    nu1: int = 1
    nu2: int = 1
    coarsest_n: int = 4
    tol: float = 1e-10
    max_iter: int = 200
    smoother: str = "vanka"
    omega: float = 24.0 / 25.0

    def orc(self) -> OrcConfig:
        return OrcConfig(0 if self.cycle == "V" else 1, self.nu1, self.nu2, self.coarsest_n, self.max_iter,
                         0 if self.smoother == "vanka" else 1, self.tol, self.omega)


class OracleError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[{status}] {msg}")
        self.status = status
        self.msg = msg


class Oracle:
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        L = self.L = C.CDLL(path)
        L.orc_last_error.restype = C.c_char_p
        L.orc_random_complex.argtypes = [C.c_uint32, C.c_double, C.c_double, C.c_int64, _dp]
        L.orc_random_real.argtypes = [C.c_uint32, C.c_double, C.c_double, C.c_int64, _dp]
        L.orc_circulant_shifts.argtypes = [C.c_double, C.c_int, C.c_double, C.c_int, C.c_int, _dp]
        L.orc_norm.restype = C.c_double
        L.orc_norm.argtypes = [C.c_int, _cp]
        L.orc_apply_shifted_laplacian.argtypes = [C.c_int, _Cplx, _cp, _cp]
        L.orc_residual.argtypes = [C.c_int, _Cplx, _cp, _cp, _cp]
        L.orc_restrict_fw.argtypes = [C.c_int, _cp, _cp]
        L.orc_prolong_bilinear.argtypes = [C.c_int, _cp, _cp]
        L.orc_vanka_coeffs.argtypes = [_Cplx, _cp, _cp, _cp]
        L.orc_jacobi_weight.argtypes = [_Cplx, C.c_double, _cp]
        L.orc_apply_smoother.argtypes = [C.c_int, _Cplx, C.c_int, C.c_double, _cp, _cp, _cp]
        L.orc_apply_stencil.argtypes = [C.c_int, _cp, C.c_double, _cp, _cp]
        L.orc_dense_operator.argtypes = [C.c_int, _Cplx, _cp]
        L.orc_dense_vanka.argtypes = [C.c_int, _Cplx, _cp]
        L.orc_mg_cycle.argtypes = [C.c_int, _Cplx, C.POINTER(OrcConfig), _cp, _cp]
        L.orc_mg_solve.argtypes = [C.c_int, _Cplx, C.POINTER(OrcConfig), _cp, _cp, _dp,
                                   C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_double)]
        L.orc_mg_solve_batch.argtypes = [C.c_int, C.c_int, _cp, C.POINTER(OrcConfig), _cp, _cp, _dp, _ip, _ip,
                                         _dp, C.c_int]
        L.orc_measured_rate.restype = C.c_double
        L.orc_measured_rate.argtypes = [_dp, C.c_int]
        L.orc_paradiag_circulant.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.POINTER(OrcConfig), _cp,
                                             _cp, _ip, _ip, C.POINTER(C.c_double), C.c_int]
        L.orc_all_at_once_residual_norm.restype = C.c_double
        L.orc_all_at_once_residual_norm.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, _cp, _cp]

    @staticmethod
    def _c(z: complex):
        return _Cplx(complex(z).real, complex(z).imag)

    def _chk(self, st: int):
        if st:
            raise OracleError(st, self.L.orc_last_error().decode())

    # inputs ------------------------------------------------------------------------------------
    def random_complex(self, seed: int, count: int, lo=-1.0, hi=1.0) -> np.ndarray:
        out = np.empty(2 * count, np.float64)
        self.L.orc_random_complex(seed, lo, hi, count, out)
        return out.view(np.complex128)

    def random_real(self, seed: int, count: int, lo=-1.0, hi=1.0) -> np.ndarray:
        out = np.empty(count, np.float64)
        self.L.orc_random_real(seed, lo, hi, count, out)
        return out

    def circulant_shifts(self, alpha: float, nt: int, dt: float, j0: int = 0, count: int | None = None):
        count = nt if count is None else count
        out = np.empty(2 * count, np.float64)
        self.L.orc_circulant_shifts(alpha, nt, dt, j0, count, out)
        return out.view(np.complex128)

    # operators (compact interior layout, shape (m, m)) ------------------------------------------
    def norm(self, n, v):
        return self.L.orc_norm(n, np.ascontiguousarray(v, np.complex128).ravel())

    def residual(self, n, lam, b, u):
        r = np.empty((n - 1) ** 2, np.complex128)
        self.L.orc_residual(n, self._c(lam), _flat(b), _flat(u), r)
        return r.reshape(n - 1, n - 1)

    def apply_shifted_laplacian(self, n, lam, u):
        r = np.empty((n - 1) ** 2, np.complex128)
        self.L.orc_apply_shifted_laplacian(n, self._c(lam), _flat(u), r)
        return r.reshape(n - 1, n - 1)

    def restrict(self, n_fine, fine):
        mc = n_fine // 2 - 1
        out = np.empty(mc * mc, np.complex128)
        self.L.orc_restrict_fw(n_fine, _flat(fine), out)
        return out.reshape(mc, mc)

    def prolong(self, n_coarse, coarse):
        mf = 2 * n_coarse - 1
        out = np.empty(mf * mf, np.complex128)
        self.L.orc_prolong_bilinear(n_coarse, _flat(coarse), out)
        return out.reshape(mf, mf)

    def vanka_coeffs(self, eta):
        a, b, c = (np.zeros(1, np.complex128) for _ in range(3))
        self._chk(self.L.orc_vanka_coeffs(self._c(eta), a, b, c))
        return complex(a[0]), complex(b[0]), complex(c[0])

    def jacobi_weight(self, eta, h):
        w = np.zeros(1, np.complex128)
        self._chk(self.L.orc_jacobi_weight(self._c(eta), h, w))
        return complex(w[0])

    def smooth(self, n, lam, u, b, kind="vanka", omega=24 / 25):
        out = np.empty((n - 1) ** 2, np.complex128)
        self._chk(self.L.orc_apply_smoother(n, self._c(lam), 0 if kind == "vanka" else 1, omega, _flat(u),
                                            _flat(b), out))
        return out.reshape(n - 1, n - 1)

    def apply_stencil(self, n, w9, scale, u):
        out = np.empty((n - 1) ** 2, np.complex128)
        self.L.orc_apply_stencil(n, np.ascontiguousarray(w9, np.complex128), scale, _flat(u), out)
        return out.reshape(n - 1, n - 1)

    def dense_operator(self, n, lam):
        N = (n - 1) ** 2
        A = np.empty(N * N, np.complex128)
        self._chk(self.L.orc_dense_operator(n, self._c(lam), A))
        return A.reshape(N, N)

    def dense_vanka(self, n, lam):
        N = (n - 1) ** 2
        M = np.empty(N * N, np.complex128)
        self._chk(self.L.orc_dense_vanka(n, self._c(lam), M))
        return M.reshape(N, N)

    def cycle(self, n, lam, cfg: Cfg, u, b):
        u = _flat(u).copy()
        oc = cfg.orc()
        self._chk(self.L.orc_mg_cycle(n, self._c(lam), C.byref(oc), u, _flat(b)))
        return u.reshape(n - 1, n - 1)

    def solve(self, n, lam, cfg: Cfg, b):
        u = np.empty((n - 1) ** 2, np.complex128)
        hist = np.zeros(cfg.max_iter + 1, np.float64)
        it, cv, rate = C.c_int(), C.c_int(), C.c_double()
        oc = cfg.orc()
        self._chk(self.L.orc_mg_solve(n, self._c(lam), C.byref(oc), _flat(b), u, hist, C.byref(it), C.byref(cv),
                                      C.byref(rate)))
        return dict(u=u.reshape(n - 1, n - 1), hist=hist[: it.value + 1].copy(), iterations=it.value,
                    converged=bool(cv.value), rate=rate.value)

    def solve_batch(self, n, lambdas, cfg: Cfg, b, threads=1):
        lam = np.ascontiguousarray(lambdas, np.complex128)
        S = lam.size
        N = (n - 1) ** 2
        b = np.ascontiguousarray(b, np.complex128).reshape(S * N)
        u = np.empty(S * N, np.complex128)
        hist = np.zeros(S * (cfg.max_iter + 1), np.float64)
        it = np.zeros(S, np.int32)
        cv = np.zeros(S, np.int32)
        rates = np.zeros(S, np.float64)
        oc = cfg.orc()
        self._chk(self.L.orc_mg_solve_batch(n, S, lam, C.byref(oc), b, u, hist, it, cv, rates, threads))
        return dict(u=u.reshape(S, n - 1, n - 1), hist=hist.reshape(S, cfg.max_iter + 1), iterations=it,
                    converged=cv.astype(bool), rates=rates)

    def paradiag(self, n, nt, alpha, dt, cfg: Cfg, f, threads=1):
        N = (n - 1) ** 2
        f = np.ascontiguousarray(f, np.complex128).reshape(nt * N)
        u = np.empty(nt * N, np.complex128)
        it = np.zeros(nt, np.int32)
        cv = np.zeros(nt, np.int32)
        rr = C.c_double()
        oc = cfg.orc()
        self._chk(self.L.orc_paradiag_circulant(n, nt, alpha, dt, C.byref(oc), f, u, it, cv, C.byref(rr), threads))
        return dict(u=u.reshape(nt, n - 1, n - 1), iterations=it, converged=cv.astype(bool), relres=rr.value)

    def all_at_once_residual_norm(self, n, nt, alpha, dt, u, f):
        return self.L.orc_all_at_once_residual_norm(n, nt, alpha, dt, _flat(u), _flat(f))


def _flat(a):
    return np.ascontiguousarray(a, np.complex128).ravel()


class RefLib:
    """The reference's own grid.cpp/smoother.cpp (+ restated driver), built under oracle/_ref."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = self.L = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_random_complex.argtypes = [C.c_uint32, C.c_double, C.c_double, C.c_int64, _dp]
        L.ref_vanka_coeffs.argtypes = [C.c_double, C.c_double, _cp]
        L.ref_apply_smoother.argtypes = [C.c_int, C.c_double, C.c_double, C.c_int, C.c_double, _cp, _cp, _cp]
        L.ref_residual.argtypes = [C.c_int, C.c_double, C.c_double, _cp, _cp, _cp]
        L.ref_apply_stencil.argtypes = [C.c_int, _cp, C.c_double, _cp, _cp]
        L.ref_restrict.argtypes = [C.c_int, _cp, _cp]
        L.ref_prolong.argtypes = [C.c_int, _cp, _cp]
        L.ref_mg_solve.argtypes = [C.c_int, C.c_double, C.c_double, _ip, _dp, _cp, _cp, _dp, C.POINTER(C.c_int),
                                   C.POINTER(C.c_int), C.POINTER(C.c_double)]
        L.ref_mg_solve_batch.argtypes = [C.c_int, C.c_int, _cp, _ip, _dp, _cp, _cp, _dp, _ip, _ip, _dp, C.c_int]

    def _chk(self, st):
        if st:
            raise OracleError(st, self.L.ref_last_error().decode())

    @staticmethod
    def _cfg(cfg: Cfg):
        ci = np.array([0 if cfg.cycle == "V" else 1, cfg.nu1, cfg.nu2, cfg.coarsest_n, cfg.max_iter,
                       0 if cfg.smoother == "vanka" else 1], np.int32)
        cd = np.array([cfg.tol, cfg.omega], np.float64)
        return ci, cd

    def random_complex(self, seed, count, lo=-1.0, hi=1.0):
        out = np.empty(2 * count, np.float64)
        self.L.ref_random_complex(seed, lo, hi, count, out)
        return out.view(np.complex128)

    def vanka_coeffs(self, eta):
        out = np.zeros(3, np.complex128)
        self._chk(self.L.ref_vanka_coeffs(complex(eta).real, complex(eta).imag, out))
        return tuple(complex(x) for x in out)

    def smooth(self, n, lam, u, b, kind="vanka", omega=24 / 25):
        out = np.empty((n - 1) ** 2, np.complex128)
        lam = complex(lam)
        self._chk(self.L.ref_apply_smoother(n, lam.real, lam.imag, 0 if kind == "vanka" else 1, omega, _flat(u),
                                            _flat(b), out))
        return out.reshape(n - 1, n - 1)

    def residual(self, n, lam, b, u):
        out = np.empty((n - 1) ** 2, np.complex128)
        lam = complex(lam)
        self._chk(self.L.ref_residual(n, lam.real, lam.imag, _flat(b), _flat(u), out))
        return out.reshape(n - 1, n - 1)

    def apply_stencil(self, n, w9, scale, u):
        out = np.empty((n - 1) ** 2, np.complex128)
        self._chk(self.L.ref_apply_stencil(n, np.ascontiguousarray(w9, np.complex128), scale, _flat(u), out))
        return out.reshape(n - 1, n - 1)

    def restrict(self, n_fine, fine):
        mc = n_fine // 2 - 1
        out = np.empty(mc * mc, np.complex128)
        self._chk(self.L.ref_restrict(n_fine, _flat(fine), out))
        return out.reshape(mc, mc)

    def prolong(self, n_coarse, coarse):
        mf = 2 * n_coarse - 1
        out = np.empty(mf * mf, np.complex128)
        self._chk(self.L.ref_prolong(n_coarse, _flat(coarse), out))
        return out.reshape(mf, mf)

    def solve(self, n, lam, cfg: Cfg, b):
        ci, cd = self._cfg(cfg)
        u = np.empty((n - 1) ** 2, np.complex128)
        hist = np.zeros(cfg.max_iter + 1, np.float64)
        it, cv, rate = C.c_int(), C.c_int(), C.c_double()
        lam = complex(lam)
        self._chk(self.L.ref_mg_solve(n, lam.real, lam.imag, ci, cd, _flat(b), u, hist, C.byref(it), C.byref(cv),
                                      C.byref(rate)))
        return dict(u=u.reshape(n - 1, n - 1), hist=hist[: it.value + 1].copy(), iterations=it.value,
                    converged=bool(cv.value), rate=rate.value)

    def solve_batch(self, n, lambdas, cfg: Cfg, b, threads=1):
        ci, cd = self._cfg(cfg)
        lam = np.ascontiguousarray(lambdas, np.complex128)
        S = lam.size
        N = (n - 1) ** 2
        u = np.empty(S * N, np.complex128)
        hist = np.zeros(S * (cfg.max_iter + 1), np.float64)
        it = np.zeros(S, np.int32)
        cv = np.zeros(S, np.int32)
        rates = np.zeros(S, np.float64)
        self._chk(self.L.ref_mg_solve_batch(n, S, lam, ci, cd, _flat(b), u, hist, it, cv, rates, threads))
        return dict(u=u.reshape(S, n - 1, n - 1), hist=hist.reshape(S, cfg.max_iter + 1), iterations=it,
                    converged=cv.astype(bool), rates=rates)
