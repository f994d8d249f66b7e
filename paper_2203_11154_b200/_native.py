"""ctypes binding of libpdmg_b200.so (the C ABI declared in include/pdmg_b200.h).

The shared library is built in-tree by `__graft_entry__.build()` (or `make -C
paper_2203_11154_b200/csrc`).  There is no fallback: if the library is missing or cannot be loaded,
importing the solver raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PDMG_B200_LIB") or os.path.join(PKG_DIR, "libpdmg_b200.so")
HEADER = os.path.join(os.path.dirname(PKG_DIR), "include", "pdmg_b200.h")

PDMG_OK, PDMG_ERR_CONFIG, PDMG_ERR_SINGULAR, PDMG_ERR_RUNTIME = 0, 1, 2, 3


class MgConfig(C.Structure):
    """pdmg_mg_config == pdmg::MultigridConfig + SmootherConfig (multigrid.hpp:14-32, smoother.hpp:30-38)."""

    _fields_ = [("cycle", C.c_int32), ("nu1", C.c_int32), ("nu2", C.c_int32), ("coarsest_n", C.c_int32),
                ("tol", C.c_double), ("max_iter", C.c_int32), ("smoother", C.c_int32), ("omega", C.c_double)]


class BatchDesc(C.Structure):
    _fields_ = [("n", C.c_int32), ("n_shifts", C.c_int32), ("lambdas", C.c_void_p), ("cfg", MgConfig),
                ("precision", C.c_int32), ("device", C.c_int32), ("devices", C.c_void_p), ("n_devices", C.c_int32)]


class C128(C.Structure):
    """pdmg_c128 (layout of std::complex<double>); passed by value in two SSE registers like the C struct."""

    _fields_ = [("re", C.c_double), ("im", C.c_double)]


class LfaConfig(C.Structure):
    _fields_ = [("samples_per_dim", C.c_int32), ("coarse_skip_tol", C.c_double)]


class SolveReport(C.Structure):
    _fields_ = [("iterations", C.c_void_p), ("converged", C.c_void_p), ("residual_history", C.c_void_p),
                ("rate", C.c_void_p), ("seconds", C.c_double)]


_lib = None


def lib() -> C.CDLL:
    """Load libpdmg_b200.so once; raise loudly if it is absent (no CPU fallback exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                          " or `make -C paper_2203_11154_b200/csrc` (the solver has no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, i32, i64, f64 = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    sig = {
        "pdmg_last_error": (C.c_char_p, []),
        "pdmg_abi_version": (C.c_int, []),
        "pdmg_mg_config_default": (None, [C.POINTER(MgConfig)]),
        "pdmg_create": (C.c_int, [C.POINTER(BatchDesc), C.POINTER(vp)]),
        "pdmg_destroy": (None, [vp]),
        "pdmg_num_levels": (C.c_int, [vp]),
        "pdmg_level_n": (C.c_int, [vp, C.c_int]),
        "pdmg_num_shifts": (C.c_int, [vp]),
        "pdmg_coarse_singular": (C.c_int, [vp, C.c_int]),
        "pdmg_solve": (C.c_int, [vp, vp, vp, C.POINTER(SolveReport)]),
        "pdmg_solve_device": (C.c_int, [vp, vp, vp, C.POINTER(SolveReport)]),
        "pdmg_solve_device_shards": (C.c_int, [vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(SolveReport)]),
        "pdmg_num_parts": (C.c_int, [vp]),
        "pdmg_part_range": (C.c_int, [vp, C.c_int, C.POINTER(i32), C.POINTER(i32), C.POINTER(i32)]),
        "pdmg_cycle": (C.c_int, [vp, vp, vp]),
        "pdmg_apply_smoother": (C.c_int, [vp, C.c_int, vp, vp, vp]),
        "pdmg_residual": (C.c_int, [vp, C.c_int, vp, vp, vp]),
        "pdmg_restrict_full_weighting": (C.c_int, [vp, C.c_int, vp, vp]),
        "pdmg_prolong_bilinear": (C.c_int, [vp, C.c_int, vp, vp]),
        "pdmg_norm": (C.c_int, [vp, C.c_int, vp, vp]),
        "pdmg_coarse_solve": (C.c_int, [vp, vp, vp]),
        "pdmg_paradiag_circulant": (C.c_int, [i32, i32, f64, f64, C.POINTER(MgConfig), i32, vp, vp,
                                              C.POINTER(SolveReport), C.POINTER(f64)]),
        "pdmg_paradiag_create": (C.c_int, [i32, i32, f64, f64, C.POINTER(MgConfig), i32, C.POINTER(vp)]),
        "pdmg_paradiag_create_multi": (C.c_int, [i32, i32, f64, f64, C.POINTER(MgConfig), vp, i32, C.POINTER(vp)]),
        "pdmg_paradiag_create_general": (C.c_int, [i32, i32, vp, vp, vp, vp, C.POINTER(MgConfig), vp, i32,
                                                   C.POINTER(vp)]),
        "pdmg_paradiag_num_parts": (C.c_int, [vp]),
        "pdmg_paradiag_part_range": (C.c_int, [vp, C.c_int, C.POINTER(i32), C.POINTER(i32), C.POINTER(i32)]),
        "pdmg_paradiag_run_shards": (C.c_int, [vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(SolveReport),
                                               C.POINTER(f64)]),
        "pdmg_paradiag_create_rank": (C.c_int, [i32, i32, f64, f64, C.POINTER(MgConfig), i32, i32, i32,
                                                C.POINTER(vp)]),
        "pdmg_paradiag_ipc_handles": (C.c_int, [vp, vp]),
        "pdmg_paradiag_open_peers": (C.c_int, [vp, vp]),
        "pdmg_paradiag_rank_phase": (C.c_int, [vp, i32, C.POINTER(SolveReport), C.POINTER(f64)]),
        "pdmg_paradiag_rank_buffer": (vp, [vp, i32]),
        "pdmg_paradiag_destroy": (None, [vp]),
        "pdmg_paradiag_solver": (vp, [vp]),
        "pdmg_paradiag_run": (C.c_int, [vp, vp, vp, C.POINTER(SolveReport), C.POINTER(f64)]),
        "pdmg_paradiag_run_device": (C.c_int, [vp, vp, vp, C.POINTER(SolveReport), C.POINTER(f64)]),
        "pdmg_time_dft": (C.c_int, [i32, i32, i64, f64, i32, vp, vp, vp]),
        "pdmg_paradiag_general": (C.c_int, [i32, i32, vp, vp, vp, vp, C.POINTER(MgConfig), i32, vp, vp,
                                            C.POINTER(SolveReport), C.POINTER(f64)]),
        "pdmg_time_transform": (C.c_int, [i32, i32, i64, vp, vp, vp, vp]),
        "pdmg_aao_residual": (C.c_int, [i32, i32, i32, i32, f64, f64, vp, vp, vp, C.POINTER(f64), vp]),
        "pdmg_lfa_config_default": (None, [C.POINTER(LfaConfig)]),
        "pdmg_lfa_symbol": (C.c_int, [i32, f64, f64, C128, f64, i32, f64, C.POINTER(C128)]),
        "pdmg_lfa_smoothing_factor": (C.c_int, [C128, f64, i32, f64, C.POINTER(LfaConfig), i32, C.POINTER(f64),
                                                C.POINTER(f64)]),
        "pdmg_lfa_smoothing_bound": (C.c_int, [C128, f64, f64, C.POINTER(LfaConfig), i32, C.POINTER(f64)]),
        "pdmg_lfa_model_create": (C.c_int, [C128, f64, i32, C.POINTER(LfaConfig), i32, C.POINTER(vp)]),
        "pdmg_lfa_model_destroy": (None, [vp]),
        "pdmg_lfa_model_skipped": (C.c_int, [vp]),
        "pdmg_lfa_model_rho": (C.c_int, [vp, i32, C.POINTER(f64), i32, C.POINTER(f64)]),
        "pdmg_lfa_model_smoothing": (C.c_int, [vp, f64, C.POINTER(f64), C.POINTER(f64)]),
        "pdmg_lfa_optimize_omega": (C.c_int, [vp, i32, i32, C.POINTER(f64), C.POINTER(f64)]),
        "pdmg_lfa_optimize_omega_smoothing": (C.c_int, [C128, f64, i32, C.POINTER(LfaConfig), i32, C.POINTER(f64),
                                                        C.POINTER(f64)]),
        "pdmg_random_rhs": (None, [C.c_uint32, f64, f64, i64, vp]),
        "pdmg_circulant_shifts": (None, [f64, i32, f64, i32, i32, vp]),
        "pdmg_host_alloc": (vp, [C.c_size_t]),
        "pdmg_host_free": (None, [vp]),
        "pdmg_stream": (vp, [vp]),
        "pdmg_set_profiling": (C.c_int, [vp, C.c_int]),
        "pdmg_set_solve_path": (C.c_int, [vp, C.c_int]),
        "pdmg_reset_stats": (None, [vp]),
        "pdmg_launch_count": (i64, [vp]),
        "pdmg_kernel_stats": (C.c_int, [vp, C.c_int, C.c_char_p, C.c_size_t, C.POINTER(i64), C.POINTER(f64),
                                        C.POINTER(f64)]),
        "pdmg_kernel_updates": (C.c_int, [vp, C.c_int, C.POINTER(f64), C.POINTER(f64)]),
        "pdmg_last_updates": (f64, [vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    if L.pdmg_abi_version() != 2:
        raise ImportError("libpdmg_b200.so ABI version mismatch")
    _lib = L
    return L


def ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def source_sha16() -> str:
    """sha256[:16] over the kernel sources (csrc/*.cuh and the Makefile with its flags, by name): the identity of the
    device code that survives a rebuild (the linked .so is not byte-reproducible) and host-only changes.
    profiles/traffic.json stamps ncu captures with it."""
    import hashlib

    d = os.path.join(PKG_DIR, "csrc")
    h = hashlib.sha256()
    for name in sorted(os.listdir(d)):
        if (name.endswith(".cuh") and name != "pdmg_engine.cuh") or name == "Makefile":
            h.update(name.encode())
            with open(os.path.join(d, name), "rb") as f:
                h.update(f.read())
    return h.hexdigest()[:16]
