"""GPU parity: every operator and full solves through the C ABI vs the CPU oracle (oracle/pdmg_oracle.c).

Tolerances (BASELINE.json north_star): complex128 solution and residual history within 1e-10 relative,
identical per-shift V-cycle counts.  Single operators agree to ~1e-14 (FMA contraction and a
re-associated 9-point sum are the only differences), checked at 1e-12.
"""
import numpy as np
import pytest

from oracle_lib import Cfg

pytestmark = pytest.mark.gpu

import paper_2203_11154_b200 as P  # noqa: E402


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    d = np.linalg.norm((a - b).ravel())
    s = np.linalg.norm(b.ravel())
    return d / s if s > 0 else d


def mgcfg(c: Cfg) -> P.MultigridConfig:
    sm = P.SmootherConfig.vanka(c.omega) if c.smoother == "vanka" else P.SmootherConfig.jacobi(c.omega)
    return P.MultigridConfig(P.CycleKind.V if c.cycle == "V" else P.CycleKind.W, c.nu1, c.nu2, c.coarsest_n, c.tol,
                             c.max_iter, sm)


LAMS = [0.0, 8.959263353215057 - 15.395328029306036j, 1000 + 1000j, -50j, 31.4 + 2j]


@pytest.mark.parametrize("n,coarsest", [(8, 4), (16, 8), (64, 4), (136, 17)])
@pytest.mark.parametrize("kind", ["vanka", "jacobi"])
def test_smoother_residual_parity(oracle, n, coarsest, kind):
    """Includes a non-power-of-two grid (136 = 8*17) whose tiles are ragged at the right/top edges."""
    cfg = Cfg(coarsest_n=coarsest, smoother=kind, omega=0.96 if kind == "vanka" else 0.8)
    m = n - 1
    S = len(LAMS)
    u = oracle.random_complex(11, S * m * m).reshape(S, m, m)
    b = oracle.random_complex(12, S * m * m).reshape(S, m, m)
    with P.BatchedMultigridHierarchy(P.Grid2D(n), LAMS, mgcfg(cfg)) as H:
        su = H.apply_smoother(0, u, b)
        r = H.residual(0, b, u)
        nr = H.norm(0, b)
    for s, lam in enumerate(LAMS):
        assert rel(su[s], oracle.smooth(n, lam, u[s], b[s], kind, cfg.omega)) < 1e-12
        assert rel(r[s], oracle.residual(n, lam, b[s], u[s])) < 1e-12
        assert abs(nr[s] - oracle.norm(n, b[s])) <= 1e-13 * oracle.norm(n, b[s])


@pytest.mark.parametrize("n", [8, 64, 256])
def test_transfer_parity(oracle, n):
    m, mc = n - 1, n // 2 - 1
    S = 3
    with P.BatchedMultigridHierarchy(P.Grid2D(n), [0.0] * S, P.MultigridConfig(coarsest_n=4)) as H:
        f = oracle.random_complex(5, S * m * m).reshape(S, m, m)
        c = oracle.random_complex(6, S * mc * mc).reshape(S, mc, mc)
        R = H.restrict_full_weighting(0, f)
        Pp = H.prolong_bilinear(0, c)
    for s in range(S):
        assert rel(R[s], oracle.restrict(n, f[s])) < 1e-14
        assert rel(Pp[s], oracle.prolong(n // 2, c[s])) < 1e-15


def test_coarse_solve_parity(oracle):
    lams = [0.0, 3 + 4j, -100j]
    with P.BatchedMultigridHierarchy(P.Grid2D(8), lams, P.MultigridConfig(coarsest_n=4)) as H:
        b = oracle.random_complex(7, 3 * 9).reshape(3, 3, 3)
        u = H.coarse_solve(b)
    for s, lam in enumerate(lams):
        r = oracle.residual(4, lam, b[s], u[s])
        assert np.linalg.norm(r) <= 1e-12 * np.linalg.norm(b[s])


@pytest.mark.parametrize("cyc", [Cfg(), Cfg(cycle="W", nu1=1, nu2=0, coarsest_n=8, tol=1e-8),
                                 Cfg(nu1=2, nu2=2), Cfg(nu1=0, nu2=2), Cfg(nu1=2, nu2=0), Cfg(nu1=3, nu2=3),
                                 Cfg(nu1=4, nu2=5, cycle="W"), Cfg(smoother="jacobi", omega=0.8)])
def test_one_cycle_parity(oracle, cyc):
    n = 64
    m = n - 1
    lams = [0.0, 8.959263353215057 - 15.395328029306036j]
    u = oracle.random_complex(21, 2 * m * m).reshape(2, m, m)
    b = oracle.random_complex(22, 2 * m * m).reshape(2, m, m)
    with P.BatchedMultigridHierarchy(P.Grid2D(n), lams, mgcfg(cyc)) as H:
        out = H.cycle(u, b)
    for s, lam in enumerate(lams):
        assert rel(out[s], oracle.cycle(n, lam, cyc, u[s], b[s])) < 1e-12


def _check_solve(oracle, n, lams, b, cfg: Cfg, tol_rel=1e-10, path="auto", expect_kernel=None):
    with P.BatchedMultigridHierarchy(P.Grid2D(n), lams, mgcfg(cfg)) as H:
        H.set_solve_path(path)
        if expect_kernel:
            H.set_profiling(True)
        u, reps = H.solve(b)
        if expect_kernel:
            names = list(H.kernel_stats())
            assert any(expect_kernel in k for k in names), names
    ref = oracle.solve_batch(n, np.asarray(lams, np.complex128), cfg, b, threads=8)
    for s in range(len(lams)):
        it = int(ref["iterations"][s])
        assert reps[s].iterations == it, (s, reps[s].iterations, it)
        assert reps[s].converged == bool(ref["converged"][s])
        hist_ref = ref["hist"][s, : it + 1]
        if hist_ref[0] == 0:  # b = 0: converged before any cycle, u = 0 exactly
            assert list(reps[s].residual_history) == [0.0] and np.all(u[s] == 0)
            continue
        assert np.max(np.abs(reps[s].residual_history - hist_ref) / hist_ref[0]) < tol_rel
        assert rel(u[s], ref["u"][s]) < tol_rel
        # rate is a geometric mean of ratios of residuals ~1e-10 r0: their roundoff differences (~1e-16 r0,
        # i.e. ~1e-6 of the last entries) carry into it
        assert abs(reps[s].rate - ref["rates"][s]) <= 1e-5 * ref["rates"][s]
    return u, reps, ref


PATHS = ["batched", "small"]


@pytest.mark.parametrize("path", PATHS)
def test_config1_single_shift(oracle, path):
    """BASELINE config 1: h=1/64, lambda_3 of the n=32 circulant family, seed 0, V(1,1), tol 1e-10."""
    lam = oracle.circulant_shifts(0.01, 32, 1 / 32, 3, 1)
    b = oracle.random_complex(0, 63 * 63).reshape(1, 63, 63)
    u, reps, ref = _check_solve(oracle, 64, lam, b, Cfg(), path=path)
    assert reps[0].iterations == 11


@pytest.mark.parametrize("path", PATHS)
def test_config2_batch32(oracle, path):
    """BASELINE config 2: h=1/128, 32 shifts, seed 1 shift-major, V(1,1): 11-12 cycles per shift."""
    lams = oracle.circulant_shifts(0.01, 32, 1 / 32)
    b = oracle.random_complex(1, 32 * 127 * 127).reshape(32, 127, 127)
    u, reps, ref = _check_solve(oracle, 128, lams, b, Cfg(), path=path)
    assert set(r.iterations for r in reps) <= {11, 12}


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("cyc", [Cfg(nu1=0, nu2=2), Cfg(nu1=2, nu2=0), Cfg(nu1=2, nu2=1, cycle="W"),
                                 Cfg(nu1=3, nu2=3), Cfg(nu1=4, nu2=2, cycle="W"),
                                 Cfg(smoother="jacobi", omega=0.8, tol=1e-8)])
def test_cycle_variants_solve(oracle, path, cyc):
    lams = oracle.circulant_shifts(0.01, 32, 1 / 32)[:3]
    b = oracle.random_complex(8, 3 * 63 * 63).reshape(3, 63, 63)
    _check_solve(oracle, 64, lams, b, cyc, path=path)


@pytest.mark.parametrize("path", PATHS)
def test_readme_w10_rates(oracle, path):
    """proj/README.md:37-41: W(1,0) at h=1/64, lambda=0: Vanka 14 cycles (0.273), Jacobi 32 (0.590)."""
    b = oracle.random_complex(123, 63 * 63).reshape(1, 63, 63)
    _, rv, _ = _check_solve(oracle, 64, [0.0], b, Cfg(cycle="W", nu1=1, nu2=0, coarsest_n=8, tol=1e-8), path=path)
    _, rj, _ = _check_solve(oracle, 64, [0.0], b, Cfg(cycle="W", nu1=1, nu2=0, coarsest_n=8, tol=1e-8,
                                                       smoother="jacobi", omega=0.8), path=path)
    assert rv[0].iterations == 14 and abs(rv[0].rate - 0.273) < 0.001
    assert rj[0].iterations == 32 and abs(rj[0].rate - 0.590) < 0.001


def test_config3_subset(oracle):
    """BASELINE config 3 shape (h=1/512, V(2,2), alpha=1e-3, dt=1/256) on 4 of its 256 shifts."""
    n, m = 512, 511
    lams = oracle.circulant_shifts(1e-3, 256, 1 / 256, 0, 256)[[0, 1, 128, 255]]
    b = oracle.random_complex(2, 4 * m * m).reshape(4, m, m)
    _check_solve(oracle, n, lams, b, Cfg(nu1=2, nu2=2))


@pytest.mark.parametrize("cyc", [Cfg(nu1=2, nu2=2), Cfg(nu1=2, nu2=2, cycle="W"), Cfg(nu1=3, nu2=4)])
def test_two_sweep_passes_ragged(oracle, cyc):
    """Levels n >= 64 run Vanka sweep pairs as one fused pass (k_march2): a non-power-of-two fine grid
    (n = 200: ragged strips at every level down to 50) on the batched path, against the oracle."""
    n, m = 200, 199
    lams = [0.0, 8.959263353215057 - 15.395328029306036j, 300 - 40j]
    b = oracle.random_complex(31, 3 * m * m).reshape(3, m, m)
    cfg = Cfg(nu1=cyc.nu1, nu2=cyc.nu2, cycle=cyc.cycle, coarsest_n=25)
    _check_solve(oracle, n, lams, b, cfg, path="batched")


@pytest.mark.parametrize("march1", ["1", "0"])
@pytest.mark.parametrize("cyc", [Cfg(nu1=1, nu2=1), Cfg(nu1=1, nu2=2), Cfg(nu1=3, nu2=1), Cfg(nu1=1, nu2=1, cycle="W"),
                                 Cfg(nu1=0, nu2=1)])
def test_single_sweep_passes_ragged(oracle, monkeypatch, cyc, march1):
    """Single Vanka sweeps on levels n >= 64 run through the marching kernel in its one-sweep form
    (k_march2<TWO = false>: sweep + restriction / norm / norm of the input iterate, prolongation + sweep);
    PDMG_MARCH1=0 routes them to the older k_level / k_march kernels.  Ragged strips (n = 200), V/W cycles
    with odd nu, against the oracle."""
    monkeypatch.setenv("PDMG_MARCH1", march1)
    n, m = 200, 199
    lams = [0.0, 8.959263353215057 - 15.395328029306036j, 300 - 40j]
    b = oracle.random_complex(32, 3 * m * m).reshape(3, m, m)
    cfg = Cfg(nu1=cyc.nu1, nu2=cyc.nu2, cycle=cyc.cycle, coarsest_n=25)
    _check_solve(oracle, n, lams, b, cfg, path="batched")


@pytest.mark.parametrize("path", PATHS)
def test_edge_cases(oracle, path):
    """multigrid test 'report edge cases' (test_multigrid.cpp:128-163) on the GPU path."""
    n = 16
    m = n - 1
    b = np.zeros((3, m, m), np.complex128)
    b[1] = oracle.random_complex(1, m * m).reshape(m, m)
    b[2] = oracle.random_complex(2, m * m).reshape(m, m)
    # shift 0: b = 0 converges at 0 iterations; others run
    cfg = Cfg(cycle="W", nu1=1, nu2=0, coarsest_n=8, tol=1e-8)
    with P.BatchedMultigridHierarchy(P.Grid2D(n), [0.0, 0.0, 0.0], mgcfg(cfg)) as H:
        H.set_solve_path(path)
        u, reps = H.solve(b)
    assert reps[0].converged and reps[0].iterations == 0 and reps[0].rate == 0.0
    assert np.all(u[0] == 0)
    assert list(reps[0].residual_history) == [0.0]
    # max_iter exhaustion reports non-convergence
    cfg2 = Cfg(cycle="W", nu1=1, nu2=0, coarsest_n=8, tol=1e-14, max_iter=1)
    with P.BatchedMultigridHierarchy(P.Grid2D(n), [0.0], mgcfg(cfg2)) as H:
        H.set_solve_path(path)
        u, reps = H.solve(b[2:3])
    assert not reps[0].converged and reps[0].iterations == 1
    h = reps[0].residual_history
    assert abs(reps[0].rate - h[1] / h[0]) < 1e-12
    # tol >= 1 converges with zero iterations
    cfg3 = Cfg(cycle="W", nu1=1, nu2=0, coarsest_n=8, tol=1.0)
    with P.BatchedMultigridHierarchy(P.Grid2D(n), [0.0], mgcfg(cfg3)) as H:
        H.set_solve_path(path)
        u, reps = H.solve(b[1:2])
    assert reps[0].converged and reps[0].iterations == 0


@pytest.mark.parametrize("path", PATHS)
def test_singular_coarse_detected(path):
    """test_multigrid.cpp:174-185: lambda = -mu_11 of the coarsest grid raises at solve."""
    cg = 8
    h = 1 / cg
    mu = (4 - 2 * np.cos(np.pi * h) - 2 * np.cos(np.pi * h)) / (h * h)
    cfg = P.MultigridConfig()
    with P.BatchedMultigridHierarchy(P.Grid2D(16), [-mu], cfg) as H:
        H.set_solve_path(path)
        assert H.coarse_singular(0)
        with pytest.raises(P.SingularOperatorError, match="singular on grid n = 8"):
            H.solve(P.random_rhs(16, 3).reshape(1, 15, 15))


@pytest.mark.parametrize("path", ["small", "batched"])
@pytest.mark.parametrize("chunks", [2, 3, 7])
def test_chunked_host_solve_matches(oracle, monkeypatch, chunks, path):
    """pdmg_solve on pinned host buffers pipelines the batch over chunks of shifts (copies overlap the
    solve); every shift's result and report must be bitwise those of the one-chunk path."""
    import ctypes

    from paper_2203_11154_b200 import _native as N

    n, S = 64, 7
    lams = [8.959263353215057 - 15.395328029306036j + 3j * k for k in range(S)]
    cfg = P.MultigridConfig(coarsest_n=4, tol=1e-10, max_iter=60)
    b = P.random_rhs(n, 5, count=S)
    with P.BatchedMultigridHierarchy(P.Grid2D(n), lams, cfg) as H:
        H.set_solve_path(path)
        u_ref, reps_ref = H.solve(b)  # pageable numpy buffers: one chunk
    monkeypatch.setenv("PDMG_IO_CHUNKS", str(chunks))
    with P.BatchedMultigridHierarchy(P.Grid2D(n), lams, cfg) as H:
        H.set_solve_path(path)
        nbytes = b.nbytes
        hb, hu = N.lib().pdmg_host_alloc(nbytes), N.lib().pdmg_host_alloc(nbytes)
        try:
            ctypes.memmove(hb, b.ctypes.data, nbytes)
            rep, it, cv, hist, rate = H._report_bufs()
            assert N.lib().pdmg_solve(H._h, hb, hu, ctypes.byref(rep)) == 0, N.lib().pdmg_last_error()
            u = np.empty_like(b)
            ctypes.memmove(u.ctypes.data, hu, nbytes)
            reps = H._reports(rep, it, cv, hist, rate)
        finally:
            N.lib().pdmg_host_free(hb)
            N.lib().pdmg_host_free(hu)
    assert np.array_equal(u, u_ref)
    for r, q in zip(reps, reps_ref):
        assert r.iterations == q.iterations and r.converged == q.converged
        assert list(r.residual_history) == list(q.residual_history)


@pytest.mark.parametrize("cyc", [Cfg(nu1=1, nu2=1, tol=1e-14, max_iter=3), Cfg(nu1=2, nu2=2, tol=1e-14, max_iter=2),
                                 Cfg(nu1=1, nu2=1, tol=1e-14, max_iter=1, smoother="jacobi", omega=0.8)])
def test_norm_next_max_iter(oracle, cyc):
    """On grids with n >= 64 the batched path forms each iterate's residual norm in the next cycle's first
    fine pass and closes the history with one norm pass after max_iter cycles; the reports (non-convergence,
    iteration counts, full history, rate) must match the oracle."""
    n, m = 128, 127
    lams = [0.0, 8.959263353215057 - 15.395328029306036j]
    b = oracle.random_complex(41, 2 * m * m).reshape(2, m, m)
    u, reps, ref = _check_solve(oracle, n, lams, b, cyc, path="batched")
    for r in reps:
        assert not r.converged and r.iterations == cyc.max_iter


def test_norm_next_mixed_convergence(oracle):
    """Shifts converging at different cycles (b = 0, an easy and a hard shift) through the norm-next path:
    a converged shift's iterate stays in the buffer its last cycle wrote while the others keep cycling."""
    n, m = 128, 127
    lams = [5000 + 0j, 0.0, 0.0, 8.959263353215057 - 15.395328029306036j]
    b = oracle.random_complex(42, 4 * m * m).reshape(4, m, m)
    b[1] = 0
    for cyc in (Cfg(nu1=1, nu2=1), Cfg(nu1=2, nu2=2), Cfg(nu1=2, nu2=2, cycle="W")):
        u, reps, ref = _check_solve(oracle, n, lams, b, cyc, path="batched")
        assert reps[1].iterations == 0 and np.all(u[1] == 0)
        assert len(set(r.iterations for r in reps)) >= 2


@pytest.mark.parametrize("pred", ["1e300", "0"])
@pytest.mark.parametrize("cyc", [Cfg(nu1=1, nu2=1), Cfg(nu1=2, nu2=2), Cfg(nu1=2, nu2=2, cycle="W"),
                                 Cfg(nu1=1, nu2=1, tol=1e-14, max_iter=6)])
def test_predicted_last_norm(oracle, monkeypatch, cyc, pred):
    """Predicted last norm (solve_device): when the host predicts that every active shift converges at
    iterate k-1, that iterate's norm comes from a residual-only pass instead of cycle k's fused first pass.
    PDMG_PRED_FINAL=1e300 forces the prediction from cycle 4 on, so most of them are wrong (the shifts
    are still far from converged, or never converge with tol 1e-14): counts, histories and iterates must
    still match the oracle; 0 disables it."""
    monkeypatch.setenv("PDMG_PRED_FINAL", pred)
    n, m = 128, 127
    lams = [5000 + 0j, 0.0, 0.0, 8.959263353215057 - 15.395328029306036j]
    b = oracle.random_complex(44, 4 * m * m).reshape(4, m, m)
    b[1] = 0
    u, reps, ref = _check_solve(oracle, n, lams, b, cyc, path="batched")
    assert reps[1].iterations == 0 and np.all(u[1] == 0)


def test_batch_beyond_coef_max(oracle):
    """A 600-shift batch on the batched path (n = 128): the marching passes take their per-shift coefficients
    as kernel parameters, COEF_MAX = 256 shifts per launch, so shifts 256..599 run in launches with
    shift0 = 256 and 512.  Every shift is checked against the oracle."""
    n, m, S = 128, 127, 600
    lams = oracle.circulant_shifts(0.01, S, 1 / 32, 0, S)
    b = oracle.random_complex(17, S * m * m).reshape(S, m, m)
    _check_solve(oracle, n, lams, b, Cfg(), path="batched")


def test_config3_sample_golden_on_gpu(oracle):
    """The reference-generated C3 sample (tests/golden/reference_golden.json, produced by the reference's own
    grid.cpp/smoother.cpp): cycle counts and residual histories within 1e-10 on the GPU path."""
    import json
    import os

    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.json")))["solves"]["C3_sample"]
    n, m = g["n"], g["n"] - 1
    lams = [complex(*x) for x in g["lambdas"]]
    b = oracle.random_complex(g["seed"], 2 * m * m).reshape(2, m, m)
    with P.BatchedMultigridHierarchy(P.Grid2D(n), lams, mgcfg(Cfg(**g["cfg"]))) as H:
        _, reps = H.solve(b)
    for j in range(2):
        h = np.array(g["hist"][j])
        assert reps[j].iterations == g["iterations"][j]
        assert np.max(np.abs(reps[j].residual_history - h) / h[0]) < 1e-10


@pytest.mark.parametrize("path", PATHS)
def test_large_coarsest_grid(oracle, path):
    """coarsest_n = 58 (57 x 57 = 3249 coarse unknowns): the batched direct solve stages 52 KB of coarse
    right-hand side in shared memory, above the 48 KB default (the kernels opt in at setup)."""
    n, m = 116, 115
    lams = [0.0, 300 - 40j]
    b = oracle.random_complex(23, 2 * m * m).reshape(2, m, m)
    _check_solve(oracle, n, lams, b, Cfg(coarsest_n=58), path=path)


def test_coarsest_too_large_is_config_error():
    """coarsest_n = 128 needs 258 KB of shared memory for the coarse right-hand side: rejected up front."""
    with pytest.raises(P.ConfigError, match="shared memory"):
        P.BatchedMultigridHierarchy(P.Grid2D(128), [0.0], P.MultigridConfig(coarsest_n=128))


@pytest.mark.parametrize("chunks", [3, 5])
def test_chunked_host_solve_marching_passes(oracle, monkeypatch, chunks):
    """The concurrent chunked host solve at n = 256 (the k_march2 / L2-prefetch passes, whose halo reads reach
    past a chunk's last shift into the next chunk's storage): bitwise the one-chunk result."""
    import ctypes

    from paper_2203_11154_b200 import _native as N

    n, m, S = 256, 255, 7
    lams = oracle.circulant_shifts(1e-3, 256, 1 / 256, 0, 256)[[0, 3, 40, 77, 128, 200, 255]]
    cfg = mgcfg(Cfg(nu1=2, nu2=2))
    b = P.random_rhs(n, 6, count=S)
    with P.BatchedMultigridHierarchy(P.Grid2D(n), lams, cfg) as H:
        u_ref, reps_ref = H.solve(b)
    monkeypatch.setenv("PDMG_IO_CHUNKS", str(chunks))
    with P.BatchedMultigridHierarchy(P.Grid2D(n), lams, cfg) as H:
        nbytes = b.nbytes
        hb, hu = N.lib().pdmg_host_alloc(nbytes), N.lib().pdmg_host_alloc(nbytes)
        try:
            ctypes.memmove(hb, b.ctypes.data, nbytes)
            rep, it, cv, hist, rate = H._report_bufs()
            assert N.lib().pdmg_solve(H._h, hb, hu, ctypes.byref(rep)) == 0, N.lib().pdmg_last_error()
            u = np.empty_like(b)
            ctypes.memmove(u.ctypes.data, hu, nbytes)
            reps = H._reports(rep, it, cv, hist, rate)
        finally:
            N.lib().pdmg_host_free(hb)
            N.lib().pdmg_host_free(hu)
    assert np.array_equal(u, u_ref)
    for r, q in zip(reps, reps_ref):
        assert r.iterations == q.iterations and list(r.residual_history) == list(q.residual_history)


@pytest.mark.gpu
@pytest.mark.parametrize("cyc,lanes,pageable", [((2, 2), 2, False), ((2, 2), 1, True), ((1, 1), 2, False), ((2, 1), 3, True)])
def test_rolling_host_solve_matches_batch(oracle, monkeypatch, cyc, lanes, pageable):
    """The rolling host solve (shifts join the batch as their right-hand sides arrive and leave it as they converge,
    each with its own cycle counter; pieces dealt to lanes that share the level arrays): bitwise the batch solve's
    iterates, identical cycle counts and residual histories, and the oracle's cycle counts (multigrid.cpp:85-110).
    Shifts with different cycle counts leave in different rounds; one right-hand side is zero (leaves at once)."""
    import ctypes

    from paper_2203_11154_b200 import _native as N

    n, S = 256, 9
    lams = np.array(oracle.circulant_shifts(1e-3, 256, 1 / 256, 0, 256))[[0, 1, 3, 40, 77, 128, 200, 254, 255]]
    lams[2], lams[6] = 1.0e6, 3.0e4 + 2.0e5j  # strongly shifted systems: fewer cycles, so they leave the batch early
    cfg = mgcfg(Cfg(nu1=cyc[0], nu2=cyc[1]))
    b = P.random_rhs(n, 8, count=S)
    b[5] = 0.0
    monkeypatch.setenv("PDMG_PRED_FINAL", "0")  # every norm of the batch solve through the same fused pass
    with P.BatchedMultigridHierarchy(P.Grid2D(n), lams, cfg) as H:
        u_ref, reps_ref = H.solve(b)
    assert len({r.iterations for r in reps_ref}) > 2
    monkeypatch.setenv("PDMG_ROLL_PIECE", "2")
    monkeypatch.setenv("PDMG_ROLL_LANES", str(lanes))
    with P.BatchedMultigridHierarchy(P.Grid2D(n), lams, cfg) as H:
        if pageable:
            u, reps = H.solve(b)
        else:
            nbytes = b.nbytes
            hb, hu = N.lib().pdmg_host_alloc(nbytes), N.lib().pdmg_host_alloc(nbytes)
            try:
                ctypes.memmove(hb, b.ctypes.data, nbytes)
                rep, it, cv, hist, rate = H._report_bufs()
                assert N.lib().pdmg_solve(H._h, hb, hu, ctypes.byref(rep)) == 0, N.lib().pdmg_last_error()
                u = np.empty_like(b)
                ctypes.memmove(u.ctypes.data, hu, nbytes)
                reps = H._reports(rep, it, cv, hist, rate)
            finally:
                N.lib().pdmg_host_free(hb)
                N.lib().pdmg_host_free(hu)
    assert np.array_equal(u, u_ref)
    for r, q in zip(reps, reps_ref):
        assert r.iterations == q.iterations and r.converged == q.converged
        assert list(r.residual_history) == list(q.residual_history)
    ref = oracle.solve_batch(n, lams, Cfg(nu1=cyc[0], nu2=cyc[1]), b, threads=8)
    assert [r.iterations for r in reps] == list(ref["iterations"])


@pytest.mark.parametrize("n,coarsest", [(72, 9), (88, 11), (104, 13), (112, 7), (144, 9), (176, 11), (208, 13), (224, 7),
                                        (288, 9), (352, 11), (416, 13), (448, 7), (576, 9)])
@pytest.mark.parametrize("cyc", [(2, 2), (1, 1)])
def test_strip_geometry_ragged_sizes(oracle, n, coarsest, cyc):
    """Edge-aligned strips of the marching passes (first strip from the ghost column, last strip ending at column m,
    1 + ceil((n - 64) / WOUT) strips per row, marched rows clamped to the domain) on level sizes that are not powers
    of two: every level of these hierarchies has a different strip count, last-strip overlap and row remainder.
    Cycle counts, histories and iterates against the oracle (multigrid.cpp:85-110)."""
    m = n - 1
    lams = oracle.circulant_shifts(1e-3, 256, 1 / 256, 0, 256)[[0, 17, 200]]
    b = oracle.random_complex(n, 3 * m * m).reshape(3, m, m)
    _check_solve(oracle, n, lams, b, Cfg(nu1=cyc[0], nu2=cyc[1], coarsest_n=coarsest), path="batched")


@pytest.mark.parametrize("S", [3, 20, 50])
def test_small_solve_cluster_matches_single_cta(oracle, monkeypatch, S):
    """The one-CTA-per-shift solve with a thread-block cluster per shift (8, 4 or 2 CTAs sharing a shift's passes,
    cluster barriers between them, the norm combined over distributed shared memory): the iterates are bitwise those
    of the single-CTA kernel, cycle counts identical, histories equal to rounding (the norm's summation order differs);
    both against the oracle (multigrid.cpp:85-110)."""
    n, m = 128, 127
    lams = oracle.circulant_shifts(0.01, 32, 1 / 32, 0, 32)[np.arange(S) % 32]
    b = oracle.random_complex(5, S * m * m).reshape(S, m, m)
    monkeypatch.setenv("PDMG_SMALL_CLUSTER", "1")
    u1, reps1, _ = _check_solve(oracle, n, lams, b, Cfg(), path="small", expect_kernel="small_solve")
    monkeypatch.setenv("PDMG_SMALL_CLUSTER", "8")
    u8, reps8, _ = _check_solve(oracle, n, lams, b, Cfg(), path="small", expect_kernel="small_solve")
    assert np.array_equal(u1, u8)
    for r1, r8 in zip(reps1, reps8):
        assert r1.iterations == r8.iterations
        assert np.allclose(r1.residual_history, r8.residual_history, rtol=1e-12, atol=0)


def test_device_list_matches_single_device(oracle):
    """One context sharded over a device list (three shards sharing GPU 0, chunks of ceil(S / 3),
    paradiag.cpp:222): host solve, device-resident shard solve, cycle and level operators are bitwise the
    single-device context's."""
    import torch

    n, m, S = 64, 63, 7
    lams = oracle.circulant_shifts(0.01, 32, 1 / 32, 0, S)
    cfg = mgcfg(Cfg())
    b = oracle.random_complex(3, S * m * m).reshape(S, m, m)
    u0 = oracle.random_complex(4, S * m * m).reshape(S, m, m)
    with P.BatchedMultigridHierarchy(P.Grid2D(n), lams, cfg) as H:
        H.set_solve_path("batched")
        u1, r1 = H.solve(b)
        c1 = H.cycle(u0, b)
        s1 = H.apply_smoother(1, u0[:, ::2, ::2][:, :31, :31].copy(), b[:, ::2, ::2][:, :31, :31].copy())
        n1 = H.norm(0, b)
    with P.BatchedMultigridHierarchy(P.Grid2D(n), lams, cfg, devices=[0, 0, 0]) as H:
        H.set_solve_path("batched")
        assert H.parts() == [(0, 3, 0), (3, 3, 0), (6, 1, 0)]
        u2, r2 = H.solve(b)
        c2 = H.cycle(u0, b)
        s2 = H.apply_smoother(1, u0[:, ::2, ::2][:, :31, :31].copy(), b[:, ::2, ::2][:, :31, :31].copy())
        n2 = H.norm(0, b)
        d_b = [torch.from_numpy(np.ascontiguousarray(b[s0:s0 + c]).view(np.float64)).cuda() for s0, c, _ in H.parts()]
        d_u = [torch.empty_like(x) for x in d_b]
        r3 = H.solve_device_shards([x.data_ptr() for x in d_b], [x.data_ptr() for x in d_u])
        torch.cuda.synchronize()
        u3 = np.concatenate([x.cpu().numpy().view(np.complex128).reshape(-1, m, m) for x in d_u])
        with pytest.raises(P.ConfigError, match="pdmg_solve_device_shards"):
            H.solve_device(d_b[0].data_ptr(), d_u[0].data_ptr())
    assert np.array_equal(u1, u2) and np.array_equal(u1, u3)
    assert np.array_equal(c1, c2) and np.array_equal(s1, s2) and np.array_equal(n1, n2)
    for a, q, w in zip(r1, r2, r3):
        assert a.iterations == q.iterations == w.iterations
        assert list(a.residual_history) == list(q.residual_history) == list(w.residual_history)


def test_device_list_bad_device_is_device_error():
    with pytest.raises(P.DeviceError, match="not available"):
        P.BatchedMultigridHierarchy(P.Grid2D(16), [0.0, 1.0], P.MultigridConfig(), devices=[0, 97])


def test_pageable_host_solve_staged_matches(oracle, monkeypatch):
    """Pageable host buffers on the chunked pipeline go through the library's pinned bounce buffers (32 MB pieces,
    multi-threaded host copies, DMA queued per piece): bitwise the plain-copy result.  83 MB per array here, so
    every direction crosses several pieces and the input ring wraps."""
    n, m, S = 512, 511, 20
    lams = oracle.circulant_shifts(1e-3, 256, 1 / 256, 0, S)
    cfg = mgcfg(Cfg(nu1=2, nu2=2))
    b = P.random_rhs(n, 7, count=S)
    monkeypatch.setenv("PDMG_IO_CHUNKS", "3")
    with P.BatchedMultigridHierarchy(P.Grid2D(n), lams, cfg) as H:
        u1, r1 = H.solve(b)  # pageable numpy arrays -> staged pipeline
    monkeypatch.setenv("PDMG_PAGEABLE", "0")
    import subprocess
    import sys
    # PDMG_PAGEABLE is read once per process: the plain-copy reference runs in a child process
    code = ("import numpy as np, sys; sys.path.insert(0, %r); import paper_2203_11154_b200 as P; "
            "lams = P.circulant_shifts(1e-3, 256, 1/256, 0, 20); "
            "cfg = P.MultigridConfig(P.CycleKind.V, 2, 2, 4, 1e-10, 200, P.SmootherConfig.vanka()); "
            "b = P.random_rhs(512, 7, count=20); H = P.BatchedMultigridHierarchy(P.Grid2D(512), lams, cfg); "
            "u, r = H.solve(b); np.save('/tmp/pdmg_plain_u.npy', u); "
            "np.save('/tmp/pdmg_plain_it.npy', np.array([x.iterations for x in r]))" % P.__path__[0].rsplit('/', 1)[0])
    subprocess.run([sys.executable, "-c", code], check=True, timeout=600)
    assert np.array_equal(u1, np.load("/tmp/pdmg_plain_u.npy"))
    assert [x.iterations for x in r1] == np.load("/tmp/pdmg_plain_it.npy").tolist()
    ref = oracle.solve_batch(n, lams[:2], Cfg(nu1=2, nu2=2), b[:2], threads=2)
    assert rel(u1[:2], ref["u"]) < 1e-10
