"""Local Fourier analysis: the numpy oracle (tests/lfa_oracle.py) pinned to the reference's published values and
known answers (CPU), and the GPU LFA (paper_2203_11154_b200.lfa over libpdmg_b200's LFA kernels) against the oracle
and the reference's own test cases (proj/tests/test_lfa.cpp, acceptance.cpp:82-139 c1-c3)."""
import math

import numpy as np
import pytest

import lfa_oracle as O

PI = math.pi


# ---- oracle pins (CPU) ----------------------------------------------------------------------------------------------
def test_oracle_reproduces_readme_table():
    """proj/README.md:108-112 / PAPER.md:136-146: the Vanka row 0.96, 0.2800, 0.2800, 0.1164, 0.0824, 0.0638 at
    h = 1/256 (unshifted; the shift of the reference's row is h^2-small)."""
    M = O.TwoGridModel(0.0, 1 / 256, "vanka")
    w, v = O.minimize_scalar(lambda w: M.rho(w, 1))
    assert round(w, 2) == 0.96 and M.skipped == 1
    assert [round(M.rho(w, nu), 4) for nu in (1, 2, 3, 4)] == [0.28, 0.1164, 0.0824, 0.0638]
    assert round(M.smoothing(w)[0], 4) == 0.28


def test_oracle_known_answers():
    """test_lfa.cpp:20-52 symbol values and the 7/25, 3/5 smoothing factors (:77-95)."""
    assert abs(O.sym_L(PI / 2, PI / 2, 0.0, 0.25) - 64.0) <= 1e-12
    assert abs(O.sym_L(0.0, 0.0, 3 - 2j, 0.25) - (3 - 2j)) <= 1e-12
    h = 0.125
    assert abs(O.sym_M(0.0, 0.0, 0.0, h, "vanka") - h * h / 2) <= 1e-15
    assert abs(O.sym_M(PI, PI, 0.0, h, "vanka") - h * h / 6) <= 1e-14
    mu, arg = O.smoothing_factor(0.0, 1 / 64, "vanka", 0.96)
    assert abs(mu - 0.28) <= 1e-10
    assert (abs(abs(arg[0]) - PI / 2) <= 1e-9 and abs(arg[1]) <= 1e-9) or \
           (abs(abs(arg[1]) - PI / 2) <= 1e-9 and abs(arg[0]) <= 1e-9)
    assert abs(O.smoothing_factor(0.0, 1 / 64, "jacobi", 0.8)[0] - 0.6) <= 1e-10


# ---- GPU LFA vs the oracle and the reference's cases ------------------------------------------------------------------
gpu = pytest.mark.gpu


@gpu
def test_symbols_and_smoothing_factor_match_oracle():
    import paper_2203_11154_b200 as P
    from paper_2203_11154_b200 import lfa

    for lam, h, kind in ((0.0, 1 / 64, "vanka"), (10 + 40j, 1 / 32, "vanka"), (5 + 15j, 1 / 32, "jacobi"),
                         (-300 + 7j, 1 / 128, "vanka")):
        cfg = P.SmootherConfig.vanka(0.9) if kind == "vanka" else P.SmootherConfig.jacobi(0.75)
        rep = lfa.smoothing_factor(lam, h, cfg)
        mu, arg = O.smoothing_factor(lam, h, kind, cfg.omega)
        assert abs(rep.mu - mu) <= 1e-13 * max(mu, 1.0)
        assert (rep.argmax.t1, rep.argmax.t2) == pytest.approx(arg, abs=1e-15)
        th = lfa.FrequencyPair(0.3, -1.1)
        assert abs(lfa.symbol_smoother_error(th, lam, h, cfg) -
                   (1 - cfg.omega * O.sym_M(0.3, -1.1, lam, h, kind) * O.sym_L(0.3, -1.1, lam, h))) <= 1e-13
    b = lfa.smoothing_factor_bound(3 + 200j, 1 / 16, 0.96)
    ob, os_ = O.smoothing_factor_bound(3 + 200j, 1 / 16, 0.96)
    assert abs(b.phi_base - ob) <= 1e-13 and abs(b.phi_shift - os_) <= 1e-13


@gpu
@pytest.mark.parametrize("lam,h,kind", [(0.0, 1 / 64, "vanka"), (0.0, 1 / 256, "jacobi"), (37j, 1 / 64, "vanka"),
                                        (120 - 90j, 1 / 32, "vanka"), (-50 + 3j, 1 / 16, "jacobi")])
def test_two_grid_model_matches_oracle(lam, h, kind):
    """rho(omega, nu) for a batch of dampings (one launch) against numpy's eigensolver on the same 4 x 4 matrices."""
    import paper_2203_11154_b200 as P
    from paper_2203_11154_b200 import lfa

    sk = P.SmootherKind.Vanka if kind == "vanka" else P.SmootherKind.Jacobi
    M = lfa.TwoGridModel(lam, h, sk)
    R = O.TwoGridModel(lam, h, kind)
    assert M.skipped_bases() == R.skipped
    ws = [0.3, 0.8, 0.96, 1.2]
    for nu in (1, 2, 4):
        got = M.rho(ws, nu)
        want = [R.rho(w, nu) for w in ws]
        np.testing.assert_allclose(got, want, rtol=1e-9, atol=1e-14)
    s = M.smoothing(0.9)
    mu, arg = R.smoothing(0.9)
    assert abs(s.mu - mu) <= 1e-13 and (s.argmax.t1, s.argmax.t2) == pytest.approx(arg, abs=1e-15)


@gpu
def test_reference_lfa_cases():
    """proj/tests/test_lfa.cpp: two-grid factors at preset damping (:117-127), the skipped null-frequency base
    (:129-137), model smoothing = standalone (:139-146), damping optimization (:148-170), config validation
    (:172-177), sampling refinement (:97-103), the shift-splitting bound over a HeatBVM family (:105-115)."""
    import paper_2203_11154_b200 as P
    from paper_2203_11154_b200 import lfa

    V, J = P.SmootherKind.Vanka, P.SmootherKind.Jacobi
    vk, jc = lfa.TwoGridModel(0.0, 1 / 256, V), lfa.TwoGridModel(0.0, 1 / 256, J)
    assert abs(vk.rho(0.96, 1) - 0.280) <= 0.005 and abs(vk.rho(0.96, 2) - 0.116) <= 0.005
    assert abs(jc.rho(0.80, 1) - 0.600) <= 0.005 and abs(jc.rho(0.80, 2) - 0.360) <= 0.005
    assert lfa.TwoGridModel(0.0, 1 / 64, V).skipped_bases() == 1
    assert lfa.TwoGridModel(37j, 1 / 64, V).skipped_bases() == 0
    m = lfa.TwoGridModel(5 + 15j, 1 / 32, V)
    assert m.smoothing(0.9).mu == pytest.approx(lfa.smoothing_factor(5 + 15j, 1 / 32, P.SmootherConfig.vanka(0.9)).mu,
                                                rel=1e-13)
    o = lfa.optimize_omega(0.0, 1 / 64, V, lfa.OmegaObjective.SmoothingMu)
    assert abs(o.omega - 0.96) <= 5e-3 and abs(o.value - 0.28) <= 1e-3
    o = lfa.optimize_omega(0.0, 1 / 64, J, lfa.OmegaObjective.SmoothingMu)
    assert abs(o.omega - 0.80) <= 5e-3 and abs(o.value - 0.60) <= 1e-3
    o = lfa.optimize_omega(lfa.TwoGridModel(0.0, 1 / 64, V), lfa.OmegaObjective.TwoGridRho, 1)
    assert abs(o.omega - 0.96) <= 0.01 and abs(o.value - 0.28) <= 0.005
    for bad in (lfa.LFAConfig(15), lfa.LFAConfig(17), lfa.LFAConfig(64, 0.0)):
        with pytest.raises(P.ConfigError):
            lfa.smoothing_factor(0.0, 0.125, P.SmootherConfig.vanka(), bad)
    with pytest.raises(P.ConfigError):
        lfa.TwoGridModel(0.0, 0.125, V, lfa.LFAConfig(10))
    s = 10 + 40j
    mu64 = lfa.smoothing_factor(s, 1 / 32, P.SmootherConfig.vanka(), lfa.LFAConfig(64)).mu
    mu128 = lfa.smoothing_factor(s, 1 / 32, P.SmootherConfig.vanka(), lfa.LFAConfig(128)).mu
    assert abs(mu64 - mu128) <= 2e-3
    td = P.TimeDiscretization(P.TimeSchemeKind.HeatBVM, 16, 1 / 16, 0.01)
    for lam in P.diagonalize_time_matrix(P.time_stepping_matrix(td)).eigenvalues:
        mu = lfa.smoothing_factor(lam, 1 / 16, P.SmootherConfig.vanka(0.96)).mu
        assert mu <= lfa.smoothing_factor_bound(lam, 1 / 16, 0.96).total() + 1e-10


@gpu
def test_acceptance_c1_c2_c3():
    """acceptance.cpp:82-139: c1 the reference table at h = tau = 1/256 (HeatBVM shift, optimized damping, mu,
    rho_nu within 0.005 / 0.01); c2 the unshifted 7/25 at 24/25 with an edge-midpoint argmax; c3 the bound
    dominates mu for every HeatBVM shift at n = 16, 64, 256."""
    import paper_2203_11154_b200 as P
    from paper_2203_11154_b200 import lfa

    def heat(n):
        td = P.TimeDiscretization(P.TimeSchemeKind.HeatBVM, n, 1.0 / n, 0.01)
        return P.diagonalize_time_matrix(P.time_stepping_matrix(td)).eigenvalues

    lam0 = heat(256)[0]
    want = {"vanka": (0.96, 0.280, [0.280, 0.116, 0.082, 0.064]), "jacobi": (0.80, 0.600, [0.600, 0.360, 0.216, 0.137])}
    for name, kind in (("vanka", P.SmootherKind.Vanka), ("jacobi", P.SmootherKind.Jacobi)):
        m = lfa.TwoGridModel(lam0, 1 / 256, kind)
        opt = lfa.optimize_omega(m, lfa.OmegaObjective.TwoGridRho, 1)
        w0, mu0, rho0 = want[name]
        assert abs(opt.omega - w0) <= 0.01
        assert abs(m.smoothing(opt.omega).mu - mu0) <= 0.005
        assert all(abs(m.rho(opt.omega, nu) - r) <= 0.005 for nu, r in zip((1, 2, 3, 4), rho0))
    rep = lfa.smoothing_factor(0.0, 1 / 64, P.SmootherConfig.vanka())
    assert abs(rep.mu - 0.28) <= 1e-10
    t1, t2 = rep.argmax.t1, rep.argmax.t2
    assert (abs(abs(t1) - PI / 2) <= 1e-9 and abs(t2) <= 1e-9) or (abs(abs(t2) - PI / 2) <= 1e-9 and abs(t1) <= 1e-9)
    for n in (16, 64, 256):
        for lam in heat(n):
            mu = lfa.smoothing_factor(lam, 1 / n, P.SmootherConfig.vanka(0.96)).mu
            assert mu <= lfa.smoothing_factor_bound(lam, 1 / n, 0.96).total() + 1e-10
