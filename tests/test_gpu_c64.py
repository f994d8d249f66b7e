"""complex64 path (BASELINE config 4 'run in both complex128 and complex64'): fp32 storage, fp64 arithmetic.
Parity target (north_star): within 1e-4 relative of the fp64 oracle; tol 1e-5 must be reached (SURVEY 0.5:
an fp32-arithmetic residual would floor at 1.2e-5)."""
import numpy as np
import pytest

from oracle_lib import Cfg

pytestmark = pytest.mark.gpu

import paper_2203_11154_b200 as P  # noqa: E402


def rel(a, b):
    return np.linalg.norm((a - b).ravel()) / np.linalg.norm(b.ravel())


def mg(c: Cfg):
    return P.MultigridConfig(P.CycleKind.V if c.cycle == "V" else P.CycleKind.W, c.nu1, c.nu2, c.coarsest_n, c.tol,
                             c.max_iter, P.SmootherConfig.vanka(c.omega))


def test_c64_operators(oracle):
    n, m = 64, 63
    lams = [0.0, 8.959 - 15.39j, 1000 + 1000j]
    u = oracle.random_complex(11, 3 * m * m).reshape(3, m, m)
    b = oracle.random_complex(12, 3 * m * m).reshape(3, m, m)
    with P.BatchedMultigridHierarchy(P.Grid2D(n), lams, P.MultigridConfig(P.CycleKind.V, 1, 1, 4),
                                     precision="c64") as H:
        su = H.apply_smoother(0, u, b)
        r = H.residual(0, b, u)
    for s, lam in enumerate(lams):
        assert rel(su[s], oracle.smooth(n, lam, u[s], b[s])) < 1e-6
        assert rel(r[s], oracle.residual(n, lam, b[s], u[s])) < 1e-6


@pytest.mark.parametrize("path", ["batched", "small"])
def test_c64_solve_config2_shape(oracle, path):
    lams = oracle.circulant_shifts(0.01, 32, 1 / 32)[:8]
    b = oracle.random_complex(1, 8 * 127 * 127).reshape(8, 127, 127)
    cfg = Cfg(tol=1e-5)
    with P.BatchedMultigridHierarchy(P.Grid2D(128), lams, mg(cfg), precision="c64") as H:
        H.set_solve_path(path)
        u, reps = H.solve(b)
    ref = oracle.solve_batch(128, lams, Cfg(tol=1e-10), b, threads=8)
    for s in range(8):
        assert reps[s].converged
        assert reps[s].residual_history[-1] <= 1e-5 * reps[s].residual_history[0]
        assert rel(u[s], ref["u"][s]) < 1e-4


def test_c64_config4_setA_small_shifts(oracle):
    """C4 set A at h=1/1024 on the smallest-|lambda| slots (j = 0, 1 of 1024, dt = 1/1024), tol 1e-5:
    the hardest case for complex64; must converge and stay within 1e-4 of fp64."""
    n, m = 1024, 1023
    lams = oracle.circulant_shifts(0.01, 1024, 1 / 1024, 0, 2)
    b = oracle.random_complex(3, 2 * m * m).reshape(2, m, m)
    with P.BatchedMultigridHierarchy(P.Grid2D(n), lams, mg(Cfg(tol=1e-5)), precision="c64") as H:
        u, reps = H.solve(b)
    with P.BatchedMultigridHierarchy(P.Grid2D(n), lams, mg(Cfg(tol=1e-10))) as H:
        u64, reps64 = H.solve(b)
    for s in range(2):
        assert reps[s].converged, reps[s].residual_history[-4:] / reps[s].residual_history[0]
        assert rel(u[s], u64[s]) < 1e-4


@pytest.mark.parametrize("cyc", [Cfg(nu1=2, nu2=2, tol=1e-5), Cfg(nu1=1, nu2=1, tol=1e-5)])
def test_c64_fused_passes(oracle, cyc):
    """complex64 through the fused two-sweep passes (V(2,2)) and the norm-next path (both), n = 256:
    the second sweep sees the fp32-stored first-sweep iterate exactly as an unfused solve would."""
    n, m = 256, 255
    lams = oracle.circulant_shifts(1e-3, 256, 1 / 256, 0, 256)[[0, 77, 200]]
    b = oracle.random_complex(5, 3 * m * m).reshape(3, m, m)
    with P.BatchedMultigridHierarchy(P.Grid2D(n), lams, mg(cyc), precision="c64") as H:
        u, reps = H.solve(b)
    ref = oracle.solve_batch(n, lams, Cfg(nu1=cyc.nu1, nu2=cyc.nu2, tol=1e-10), b, threads=8)
    for s in range(3):
        assert reps[s].converged
        assert reps[s].residual_history[-1] <= 1e-5 * reps[s].residual_history[0]
        assert rel(u[s], ref["u"][s]) < 1e-4
