"""CPU tests: pin the oracle (oracle/pdmg_oracle.c) against the reference's own outputs and known answers.

tests/golden/reference_golden.json was produced by the reference's unmodified grid.cpp/smoother.cpp
(tests/golden/make_golden.py); the oracle restates the same floating-point operation order, so operators
and solves must match BIT-FOR-BIT.  The known-answer tests restate the reference's own unit tests
(proj/tests/test_grid.cpp, test_smoother.cpp, test_multigrid.cpp) against the oracle.
"""
import json
import os

import numpy as np
import pytest

from oracle_lib import Cfg, OracleError

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.json")))


def l2c(x):
    a = np.asarray(x, np.float64)
    return a[..., 0] + 1j * a[..., 1]


def test_rng_matches_reference_stream(oracle):
    """std::mt19937 + uniform_real_distribution<double>(-1,1), re then im (tools/pdmg.cpp:137-147)."""
    for seed, vals in GOLD["rng"].items():
        assert np.array_equal(oracle.random_complex(int(seed), len(vals)), l2c(vals))


@pytest.mark.parametrize("k", range(3))
def test_operators_bit_identical(oracle, k):
    g = GOLD["operators"][k]
    n, lam = g["n"], complex(*g["lambda"])
    m, mc = n - 1, n // 2 - 1
    u = oracle.random_complex(g["u_seed"], m * m).reshape(m, m)
    b = oracle.random_complex(g["b_seed"], m * m).reshape(m, m)
    c = oracle.random_complex(g["c_seed"], mc * mc).reshape(mc, mc)
    assert np.array_equal(oracle.smooth(n, lam, u, b, "vanka", 24 / 25).ravel(), l2c(g["vanka"]))
    assert np.array_equal(oracle.smooth(n, lam, u, b, "jacobi", 4 / 5).ravel(), l2c(g["jacobi"]))
    assert np.array_equal(oracle.residual(n, lam, b, u).ravel(), l2c(g["residual"]))
    assert np.array_equal(oracle.restrict(n, u).ravel(), l2c(g["restrict"]))
    assert np.array_equal(oracle.prolong(n // 2, c).ravel(), l2c(g["prolong"]))


def test_vanka_coeffs_bit_identical(oracle):
    for e in GOLD["vanka_coeffs"]:
        got = oracle.vanka_coeffs(complex(*e["eta"]))
        assert np.array_equal(np.array(got), l2c(e["abc"]))


def _cfg(d):
    return Cfg(**d)


@pytest.mark.parametrize("name", ["C1", "W10_vanka", "W10_jacobi"])
def test_single_solves_bit_identical(oracle, name):
    g = GOLD["solves"][name]
    n = g["n"]
    b = oracle.random_complex(g["seed"], (n - 1) ** 2).reshape(n - 1, n - 1)
    s = oracle.solve(n, complex(*g["lambda"]), _cfg(g["cfg"]), b)
    assert s["iterations"] == g["iterations"]
    assert np.array_equal(s["hist"], np.array(g["hist"]))
    assert s["rate"] == g["rate"]
    if "u" in g:
        u = s["u"].ravel()
        assert np.array_equal(u[:4], l2c(g["u"]["first"]))
        assert float(np.sum(np.abs(u) ** 2)) == pytest.approx(g["u"]["sumsq"], rel=1e-15)


def test_readme_rates(oracle):
    """proj/README.md:37-41: Vanka W(1,0) 14 cycles at ~0.273, Jacobi 32 at ~0.590."""
    assert GOLD["solves"]["W10_vanka"]["iterations"] == 14
    assert abs(GOLD["solves"]["W10_vanka"]["rate"] - 0.273) < 1e-3
    assert GOLD["solves"]["W10_jacobi"]["iterations"] == 32
    assert abs(GOLD["solves"]["W10_jacobi"]["rate"] - 0.590) < 1e-3


def test_config2_batch_matches_reference(oracle):
    g = GOLD["solves"]["C2"]
    lams = l2c(g["lambdas"])
    b = oracle.random_complex(1, 32 * 127 * 127).reshape(32, 127, 127)
    s = oracle.solve_batch(128, lams, _cfg(g["cfg"]), b, threads=8)
    assert s["iterations"].tolist() == g["iterations"]
    for j in range(32):
        it = g["iterations"][j]
        assert np.array_equal(s["hist"][j, : it + 1], np.array(g["hist"][j]))
        assert np.array_equal(s["u"][j].ravel()[:4], l2c(g["u"][j]["first"]))


def test_config3_sample_matches_reference(oracle):
    """BASELINE config 3 shape (h=1/512, V(2,2), alpha=1e-3): the reference-generated C3 sample (slots 0 and 128
    with the first two seed-2 right-hand sides, tests/golden/make_golden.py) -- cycle counts and residual
    histories bit for bit."""
    g = GOLD["solves"]["C3_sample"]
    n, m = g["n"], g["n"] - 1
    lams = l2c(g["lambdas"])
    b = oracle.random_complex(g["seed"], 2 * m * m).reshape(2, m, m)
    s = oracle.solve_batch(n, lams, _cfg(g["cfg"]), b, threads=2)
    for j in range(2):
        it = g["iterations"][j]
        assert s["iterations"][j] == it
        assert np.array_equal(s["hist"][j, : it + 1], np.array(g["hist"][j]))


def test_banded_coarse_factor_large_coarsest(oracle):
    """The coarsest-level LU (dense.cpp:82-100) exploits the band of A + lambda I (skipping exact zeros only):
    a 57 x 57 coarsest grid (3249 unknowns) factors quickly and solves to roundoff."""
    n = 58
    m = n - 1
    for lam in (0.0, 300 - 40j):
        b = oracle.random_complex(9, m * m).reshape(m, m)
        s = oracle.solve(n, lam, Cfg(coarsest_n=n, nu1=1, nu2=1), b)  # single level: a direct solve
        assert s["iterations"] == 1 and s["converged"]
        r = oracle.residual(n, lam, b, s["u"])
        assert np.linalg.norm(r) <= 1e-10 * np.linalg.norm(b)


def test_threads_bitwise_identical(oracle):
    """paradiag test 'multi-threaded result is bitwise identical' (test_paradiag.cpp:250-259)."""
    lams = oracle.circulant_shifts(0.01, 32, 1 / 32)[:6]
    b = oracle.random_complex(5, 6 * 31 * 31).reshape(6, 31, 31)
    a1 = oracle.solve_batch(32, lams, Cfg(), b, threads=1)
    a3 = oracle.solve_batch(32, lams, Cfg(), b, threads=3)
    assert np.array_equal(a1["u"], a3["u"]) and np.array_equal(a1["hist"], a3["hist"])


def test_baseline_shift_formula(oracle):
    """C1's shift: lambda_3 of alpha=0.01, n=32, dt=1/32: (8.95926, -15.3953)."""
    lam = oracle.circulant_shifts(0.01, 32, 1 / 32, 3, 1)[0]
    assert abs(lam - (8.959263353215057 - 15.395328029306036j)) < 1e-12
    assert complex(*GOLD["solves"]["C1"]["lambda"]) == lam


# ---------------- known answers restated from the reference's unit tests ----------------------------
def test_vanka_coeff_known_answers(oracle):
    a, b, c = oracle.vanka_coeffs(0.0)  # test_smoother.cpp:14-19
    assert abs(a - 7 / 24) <= 1e-15 and abs(b - 1 / 12) <= 1e-15 and abs(c - 1 / 24) <= 1e-15
    for eta in (0.1, 1 + 1j, -0.5j, -1 + 3j):  # :21-28
        a, b, c = oracle.vanka_coeffs(eta)
        assert abs((a + 2 * b + c) - 1 / (2 + eta)) <= 1e-13
        assert abs((a - 2 * b + c) - 1 / (6 + eta)) <= 1e-13
        assert abs((a - c) - 1 / (4 + eta)) <= 1e-13


def test_singular_rejection(oracle):
    for eta in (-2.0, -4.0, -6.0, -2 + 1e-15j):  # test_smoother.cpp:30-39
        with pytest.raises(OracleError) as e:
            oracle.vanka_coeffs(eta)
        assert e.value.status == 2
    oracle.vanka_coeffs(-2 + 0.1j)
    with pytest.raises(OracleError):
        oracle.jacobi_weight(-4.0, 0.1)
    assert abs(oracle.jacobi_weight(0.0, 0.5) - 0.0625) <= 1e-15


@pytest.mark.parametrize("lam", [0.0, 10.0, 100 + 100j, -50j])
def test_stencil_equals_patch_sum(oracle, lam):
    """closed-form stencil == assembled patch sum incl. boundary rows (test_smoother.cpp:64-79)."""
    n = 10
    m = n - 1
    M = oracle.dense_vanka(n, lam)
    u = oracle.random_complex(77, m * m)
    w = np.zeros(9, np.complex128)
    a, b, c = oracle.vanka_coeffs(lam / n ** 2)
    w[:] = [c, 2 * b, c, 2 * b, 4 * a, 2 * b, c, 2 * b, c]
    mu = oracle.apply_stencil(n, w, (1 / n) ** 2 / 4, u).ravel()
    assert np.max(np.abs(M @ u - mu)) <= 1e-13


def test_smoother_fixed_point_and_error_propagation(oracle):
    n, m = 8, 7
    lam = 5 + 2j  # test_smoother.cpp:81-92
    ustar = oracle.random_complex(9, m * m).reshape(m, m)
    b = oracle.apply_shifted_laplacian(n, lam, ustar)
    for kind, om in (("vanka", 0.96), ("jacobi", 0.8)):
        u1 = oracle.smooth(n, lam, ustar, b, kind, om)
        assert np.linalg.norm(u1 - ustar) <= 1e-12 * np.linalg.norm(ustar)
    lam = 2 - 3j  # :94-120
    A = oracle.dense_operator(n, lam)
    E = np.eye(m * m) - 0.9 * oracle.dense_vanka(n, lam) @ A
    u = oracle.random_complex(21, m * m)
    su = oracle.smooth(n, lam, u.reshape(m, m), np.zeros((m, m)), "vanka", 0.9).ravel()
    assert np.linalg.norm(E @ u - su) <= 1e-12 * np.linalg.norm(E @ u)


def test_grid_known_answers(oracle):
    # restriction of the values 1..9 around a coarse node is 5 (test_grid.cpp:143-158)
    n = 4
    f = np.arange(1, 10, dtype=np.complex128).reshape(3, 3)
    assert oracle.restrict(n, f)[0, 0] == 5.0
    # prolongation tent (test_grid.cpp:160-178)
    c = np.zeros((3, 3), np.complex128)
    c[1, 1] = 1.0
    p = oracle.prolong(4, c)
    assert p[3, 3] == 1.0 and p[3, 2] == 0.5 and p[2, 2] == 0.25 and p[1, 1] == 0.0
    # R = (1/4) P^T (test_grid.cpp:180-190)
    nf, mf, mc = 8, 7, 3
    P = np.stack([oracle.prolong(4, np.eye(mc * mc)[k].reshape(mc, mc)).ravel() for k in range(mc * mc)], axis=1)
    R = np.stack([oracle.restrict(nf, np.eye(mf * mf)[k].reshape(mf, mf)).ravel() for k in range(mf * mf)], axis=1)
    assert np.max(np.abs(R - 0.25 * P.T)) < 1e-15
    # sine eigenfunctions (test_grid.cpp:59-83)
    n = 16
    h = 1 / n
    i = np.arange(1, n)
    for p_, q_ in ((1, 1), (3, 5)):
        u = np.outer(np.sin(q_ * np.pi * i * h), np.sin(p_ * np.pi * i * h)).astype(np.complex128)
        ev = (4 - 2 * np.cos(p_ * np.pi * h) - 2 * np.cos(q_ * np.pi * h)) / h ** 2
        Au = oracle.apply_shifted_laplacian(n, 0.0, u)
        assert np.max(np.abs(Au - ev * u)) <= 1e-10 * ev


def test_multigrid_edge_cases(oracle):
    cfg = Cfg(cycle="W", nu1=1, nu2=0, coarsest_n=8, tol=1e-8)  # test_multigrid.cpp:128-163
    z = np.zeros((15, 15), np.complex128)
    s = oracle.solve(16, 0.0, cfg, z)
    assert s["converged"] and s["iterations"] == 0 and s["rate"] == 0.0 and list(s["hist"]) == [0.0]
    b = oracle.random_complex(2, 225).reshape(15, 15)
    s = oracle.solve(16, 0.0, Cfg(cycle="W", nu1=1, nu2=0, coarsest_n=8, tol=1e-14, max_iter=1), b)
    assert not s["converged"] and s["iterations"] == 1 and len(s["hist"]) == 2
    assert s["rate"] == pytest.approx(s["hist"][1] / s["hist"][0], rel=1e-12)
    s = oracle.solve(16, 0.0, Cfg(cycle="W", nu1=1, nu2=0, coarsest_n=8, tol=1.0), b)
    assert s["converged"] and s["iterations"] == 0
    # V is no faster than W (test_multigrid.cpp:187-198)
    b = oracle.random_complex(17, 31 * 31).reshape(31, 31)
    w = oracle.solve(32, 0.0, Cfg(cycle="W", nu1=1, nu2=0, coarsest_n=8, tol=1e-8), b)
    v = oracle.solve(32, 0.0, Cfg(cycle="V", nu1=1, nu2=0, coarsest_n=8, tol=1e-8), b)
    assert v["iterations"] >= w["iterations"]


def test_hierarchy_validation_messages(oracle):
    with pytest.raises(OracleError, match="reaches n = 4, not coarsest_n = 5"):
        oracle.solve(64, 0.0, Cfg(coarsest_n=5), np.zeros((63, 63)))
    with pytest.raises(OracleError, match=r"level 0 \(n = 64\): vanka_coeffs"):
        oracle.solve(64, -2 * 64 * 64, Cfg(), np.ones((63, 63)))
    cg = 8
    mu = (4 - 4 * np.cos(np.pi / cg)) * cg * cg  # test_multigrid.cpp:174-185
    with pytest.raises(OracleError, match="singular on grid n = 8") as e:
        oracle.solve(16, -mu, Cfg(cycle="W", nu1=1, nu2=0, coarsest_n=8, tol=1e-8),
                     oracle.random_complex(3, 225).reshape(15, 15))
    assert e.value.status == 2


def test_paradiag_circulant_small(oracle):
    """alpha-circulant ParaDIAG restatement: the all-at-once residual of the C_alpha system is at the
    multigrid tolerance (exact inner solves would give ~1e-15)."""
    n, nt = 16, 8
    m = n - 1
    f = oracle.random_complex(4, nt * m * m).reshape(nt, m, m)
    r = oracle.paradiag(n, nt, 0.01, 1 / nt, Cfg(tol=1e-12), f, threads=4)
    assert r["converged"].all()
    assert r["relres"] < 1e-10


def test_qbv_scheme_matches_dense_kronecker(oracle):
    """'space-time solve with the regularized backward scheme matches its oracle' (test_paradiag.cpp:214-226):
    BackwardHeatQBV = alpha-circulant with alpha = -1/beta; tiny grid so the coarse solve is exact."""
    import numpy as np

    import paper_2203_11154_b200 as P

    td = P.TimeDiscretization(P.TimeSchemeKind.BackwardHeatQBV, 4, 0.25, 0.01)
    n, m, nt = 4, 3, td.dim()
    B = P.time_stepping_matrix(td)
    K = np.kron(B, np.eye(m * m)) + np.kron(np.eye(nt), oracle.dense_operator(n, 0.0))
    f = np.stack([oracle.random_complex(50 + i, m * m) for i in range(nt)])
    want = np.linalg.solve(K, f.ravel())
    r = oracle.paradiag(n, nt, td.circulant_alpha(), td.tau, Cfg(coarsest_n=4), f, threads=2)
    assert np.linalg.norm(r["u"].ravel() - want) <= 1e-8 * np.linalg.norm(want)
    assert r["relres"] <= 1e-10
    # the closed-form eigenvalues (paradiag.cpp:221) are the shift set, in reversed slot order
    g = (1 / td.beta) ** (1 / nt) * np.exp(1j * np.pi / nt)
    ref = np.array([(1 - g * np.exp(-2j * np.pi * k / nt)) / td.tau for k in range(nt)])
    mine = oracle.circulant_shifts(td.circulant_alpha(), nt, td.tau)
    np.testing.assert_allclose(mine, ref[(-np.arange(nt)) % nt], rtol=1e-13)
