"""paper_2203_11154_b200 -- B200-native batched complex-shifted-Laplacian multigrid (Vanka V-cycles).

Host mirror of the reference `pdmg` solver interface over libpdmg_b200.so (sm_100a CUDA + C ABI,
include/pdmg_b200.h).  See DESIGN.md.
"""
from .multigrid import (BatchedMultigridHierarchy, ConfigError, CycleKind, DeviceError, Grid2D, MultigridConfig,
                        MultigridHierarchy, Shift, ShiftKind, SingularOperatorError, SmootherConfig, SmootherKind,
                        SolveReport, circulant_shifts, multigrid_solve, random_rhs)

from .paradiag import (ParadiagCirculant, ParadiagGeneral, TimeDiagonalization, TimeDiscretization, TimeSchemeKind,  # noqa: E402
                       all_at_once_apply, diagonalize_qbv_closed_form, diagonalize_time_matrix, helmholtz_shifts,
                       manufactured_field,
                       paradiag_solve, time_stepping_matrix)

from . import lfa  # noqa: E402

__all__ = [
    "lfa",
    "ParadiagCirculant", "ParadiagGeneral", "diagonalize_qbv_closed_form", "TimeDiagonalization", "TimeDiscretization", "TimeSchemeKind", "all_at_once_apply",
    "diagonalize_time_matrix", "helmholtz_shifts", "manufactured_field", "paradiag_solve", "time_stepping_matrix",
    "BatchedMultigridHierarchy", "ConfigError", "CycleKind", "DeviceError", "Grid2D", "MultigridConfig",
    "MultigridHierarchy", "Shift", "ShiftKind", "SingularOperatorError", "SmootherConfig", "SmootherKind",
    "SolveReport", "circulant_shifts", "multigrid_solve", "random_rhs",
]
