"""BASELINE config 4 at full size against the CPU oracle: 1024 shifts at h = 1/1024 (1023 x 1023 interior), V(1,1),
seed-3 right-hand sides drawn shift-major, both shift sets (A: dt = 1/1024; B: dt = h^2, whose slot j = 512 has
eta = lambda h^2 = 2), in complex128 (tol 1e-10) and complex64 (tol 1e-5).

The whole 1024-shift batch runs on the GPU in one context, so every launch covers shift ranges past the first
COEF_MAX = 256 (the multi-launch coefficient packs with shift0 > 0, pdmg_capi.cu level_pass2).  The oracle
(oracle/pdmg_oracle.c, restating proj/src/multigrid.cpp:85-110) solves a sample of slots on both sides of every
256-shift boundary: identical cycle counts, solution and residual history within 1e-10 relative (c128), and
within 1e-4 of the fp64 oracle for complex64 (north_star tolerances).
"""
import numpy as np
import pytest

from oracle_lib import Cfg

pytestmark = pytest.mark.gpu

import paper_2203_11154_b200 as P  # noqa: E402

N_GRID, S = 1024, 1024
SAMPLE = [0, 1, 255, 256, 257, 511, 512, 767, 1023]
SETS = {"A": 1.0 / 1024, "B": 2.0 ** -20}


def rel(a, b):
    return np.linalg.norm((a - b).ravel()) / np.linalg.norm(b.ravel())


@pytest.fixture(scope="module")
def c4():
    import torch

    m = N_GRID - 1
    b = P.random_rhs(N_GRID, 3, count=S)  # one mt19937(3) stream, shift-major: 17.1 GB
    d_b = torch.from_numpy(b.view(np.float64)).to("cuda:0")
    d_u = torch.empty_like(d_b)
    sample_b = np.ascontiguousarray(b[SAMPLE])
    del b
    yield dict(m=m, d_b=d_b, d_u=d_u, sample_b=sample_b, oracle={})
    del d_b, d_u
    torch.cuda.empty_cache()


def _oracle(oracle, c4, name):
    if name not in c4["oracle"]:
        lams = P.circulant_shifts(0.01, 1024, SETS[name], 0, S)[SAMPLE]
        c4["oracle"][name] = oracle.solve_batch(N_GRID, lams, Cfg(nu1=1, nu2=1), c4["sample_b"], threads=len(SAMPLE))
    return c4["oracle"][name]


def _gpu(c4, name, precision):
    import torch

    lams = P.circulant_shifts(0.01, 1024, SETS[name], 0, S)
    tol = 1e-10 if precision == "c128" else 1e-5
    cfg = P.MultigridConfig(P.CycleKind.V, 1, 1, 4, tol, 200, P.SmootherConfig.vanka())
    with P.BatchedMultigridHierarchy(P.Grid2D(N_GRID), lams, cfg, precision=precision) as H:
        reps = H.solve_device(c4["d_b"].data_ptr(), c4["d_u"].data_ptr())
    torch.cuda.synchronize()
    u = c4["d_u"].view(S, c4["m"], c4["m"], 2)[SAMPLE].cpu().numpy()
    return reps, (u[..., 0] + 1j * u[..., 1])


@pytest.mark.parametrize("name", ["A", "B"])
def test_config4_c128_matches_oracle(oracle, c4, name):
    reps, u = _gpu(c4, name, "c128")
    assert all(r.converged for r in reps)
    ref = _oracle(oracle, c4, name)
    margins = []
    for q, j in enumerate(SAMPLE):
        it = int(ref["iterations"][q])
        assert reps[j].iterations == it, (j, reps[j].iterations, it)
        h_ref = ref["hist"][q, : it + 1]
        assert np.max(np.abs(reps[j].residual_history - h_ref) / h_ref[0]) < 1e-10
        assert rel(u[q], ref["u"][q]) < 1e-10
        margins.append(abs(h_ref[-1] / h_ref[0] - 1e-10) / 1e-10)
    if name == "B":  # slot 512: eta = 2 on the fine grid, the easiest shift of set B (8 cycles)
        assert reps[512].iterations < reps[0].iterations
    print(f"C4 set {name} c128: sampled cycles {[reps[j].iterations for j in SAMPLE]}, "
          f"all cycles {sorted(set(r.iterations for r in reps))}, min stop margin {min(margins):.3g}")


@pytest.mark.parametrize("name", ["A", "B"])
def test_config4_c64_within_1e4_of_oracle(oracle, c4, name):
    reps, u = _gpu(c4, name, "c64")
    ref = _oracle(oracle, c4, name)
    for r in reps:
        assert r.converged and r.residual_history[-1] <= 1e-5 * r.residual_history[0]
    for q, j in enumerate(SAMPLE):
        assert rel(u[q], ref["u"][q]) < 1e-4, (j, rel(u[q], ref["u"][q]))
