"""CLI driver (paper_2203_11154_b200/cli.py): runio known answers (proj/tests/test_runio.cpp), usage errors and
exit codes on CPU, and real solve/sweep/paradiag runs on the GPU (proj/tests/test_cli.cpp shapes)."""
import io
import math
import subprocess
import sys

import numpy as np
import pytest

from paper_2203_11154_b200 import cli
from paper_2203_11154_b200.multigrid import ConfigError


def test_parse_reciprocal_known_answers():
    for s, v in (("1/256", 256), ("1/2", 2), ("1/3", 3), ("2/512", 256), ("0.00390625", 256), ("0.25", 4),
                 ("0.333333333333333", 3)):
        assert cli.parse_reciprocal(s) == v
    for bad in ("abc", "1/0", "0", "-1/4", "2/3", "0.3", "1", "1/4x", ""):
        with pytest.raises(ConfigError):
            cli.parse_reciprocal(bad)


def test_format_and_fnv1a():
    assert cli.format_sig(0.28) == "0.28" and cli.format_sig(1.0) == "1"
    assert cli.format_sig(math.pi) == "3.14159265358979"
    assert cli.fnv1a_hex("") == "cbf29ce484222325"
    assert cli.fnv1a_hex("a") == "af63dc4c8601ec8c"
    assert cli.fnv1a_hex("foobar") == "85944171f73967e8"


def test_manifest_and_csv_shape():
    m = cli.RunManifest("solve")
    m.add("h", "1/64")
    h1 = cli.fnv1a_hex(m.canonical())
    m2 = cli.RunManifest("solve")
    m2.add("h", "1/32")
    assert cli.fnv1a_hex(m2.canonical()) != h1
    buf = io.StringIO()
    w = cli.CsvWriter(buf, m, ["iter", "residual"])
    w.row(["0", "1"])
    with pytest.raises(ConfigError):
        w.row(["0"])
    lines = buf.getvalue().splitlines()
    assert lines[0] == f"# pdmg solve v{cli.VERSION}" and lines[1] == f"# manifest-hash: {h1}"
    assert lines[2] == "# h = 1/64" and lines[3] == "iter,residual" and lines[4] == "0,1"


def test_qbv_eigenvalues_closed_form():
    """paradiag.cpp:219-221: (1 - gamma zeta^{-k}) / tau equals the eigenvalues of the dense QBV matrix."""
    from paper_2203_11154_b200.paradiag import TimeDiscretization, TimeSchemeKind, time_stepping_matrix

    lam = cli.qbv_eigenvalues(6, 1 / 6, 0.01)
    ev = np.linalg.eigvals(time_stepping_matrix(TimeDiscretization(TimeSchemeKind.BackwardHeatQBV, 6, 1 / 6, 0.01)))
    for z in lam:
        assert np.min(np.abs(ev - z)) <= 1e-9 * abs(z)


@pytest.mark.parametrize("argv", [
    ["solve"],                                      # missing --h
    ["solve", "--h", "1/3x"],                       # malformed fraction
    ["solve", "--h", "1/64", "--h0", "1/5"],        # coarsening mismatch (ConfigError before any CUDA call)
    ["solve", "--h", "1/64", "--scheme", "helmholtz", "--lambda-re", "1"],
    ["sweep", "--h", "1/16", "--example", "heat", "--smoothers", "foo"],
    ["paradiag", "--h", "1/16", "--threads", "0"],
])
def test_usage_errors_exit_1(argv):
    assert cli.main(argv) == 1


def _run(args):
    return subprocess.run([sys.executable, "-m", "paper_2203_11154_b200"] + args, capture_output=True, text=True,
                          timeout=300)


@pytest.mark.gpu
def test_cli_solve_config1():
    r = _run(["solve", "--h", "1/64", "--lambda-re", "8.959263353215057", "--lambda-im", "-15.395328029306036",
              "--cycle", "v", "--nu1", "1", "--nu2", "1", "--h0", "1/4", "--tol", "1e-10", "--seed", "0"])
    assert r.returncode == 0, r.stderr
    rows = [ln for ln in r.stdout.splitlines() if ln and not ln.startswith("#")]
    assert rows[0] == "iter,residual" and len(rows) == 13  # header + residual history of 11 cycles
    res = [float(x.split(",")[1]) for x in rows[1:]]
    assert res[-1] <= 1e-10 * res[0] and "iterations=11" in r.stderr


@pytest.mark.gpu
def test_cli_sweep_and_paradiag():
    r = _run(["sweep", "--example", "backward-heat", "--h", "1/32", "--tau", "1/8"])
    assert r.returncode == 0, r.stderr
    rows = [ln for ln in r.stdout.splitlines() if ln and not ln.startswith("#")]
    assert rows[0].startswith("shift_index,lambda_re") and len(rows) == 1 + 2 * 9
    assert all(ln.split(",")[6] == "true" for ln in rows[1:])
    for scheme in ("heat-bvm", "backward-heat"):
        r = _run(["paradiag", "--scheme", scheme, "--h", "1/16"])
        assert r.returncode == 0, r.stderr
        assert "all_converged=true" in r.stderr
        err = float(r.stderr.split("manufactured_error=")[1].split()[0])
        assert err <= 1e-5


def _rows(out):
    return [ln for ln in out.splitlines() if ln and not ln.startswith("#")]


@pytest.mark.gpu
def test_cli_reference_cases():
    """proj/tests/test_cli.cpp cases on the GPU backend: usage errors, help/version, solve CSV + manifest and its
    byte-identical rerun (:96-99), scheme-derived shift with a manufactured rhs, file output, the singular coarse
    shift (exit 2), sweep shapes, paradiag and its non-convergence exit code."""
    for args in ([], ["frobnicate"], ["solve", "--h", "1/16", "--smoother", "sor"], ["sweep", "--h", "1/16"],
                 ["solve", "--h", "1/16", "--scheme", "heat-bvm", "--shift-index", "99"]):
        assert cli.main(args) == 1, args
    r = _run(["--version"])
    assert r.returncode == 0 and "pdmg" in r.stdout
    r = _run(["solve", "--h", "1/16", "--lambda-re", "2", "--lambda-im", "3"])
    assert r.returncode == 0, r.stderr
    assert "# pdmg solve v" in r.stdout and "# manifest-hash: " in r.stdout and "iter,residual" in r.stdout
    rows = _rows(r.stdout)
    assert len(rows) >= 3 and rows[1].startswith("0,") and "converged=true" in r.stderr
    again = _run(["solve", "--h", "1/16", "--lambda-re", "2", "--lambda-im", "3"])
    assert again.stdout == r.stdout  # stdout is deterministic across runs
    r = _run(["solve", "--h", "1/16", "--scheme", "heat-bvm", "--tau", "1/16", "--shift-index", "1", "--rhs",
              "manufactured"])
    assert r.returncode == 0 and "lambda_im" in r.stdout and "converged=true" in r.stderr
    path = "/tmp/pdmg_b200_cli_test.csv"
    r = _run(["solve", "--h", "1/16", "--out", path])
    assert r.returncode == 0 and r.stdout == "" and "iter,residual" in open(path).read()
    h = 0.125
    mu = (4.0 - 4.0 * math.cos(math.pi * h)) / (h * h)
    r = _run(["solve", "--h", "1/8", "--lambda-re", repr(-mu)])
    assert r.returncode == 2 and "singular" in r.stderr
    r = _run(["sweep", "--example", "heat", "--h", "1/16", "--tau", "1/16"])
    assert r.returncode == 0 and len(_rows(r.stdout)) == 1 + 32
    assert all(",true," in ln for ln in _rows(r.stdout)[1:])
    r = _run(["sweep", "--example", "helmholtz", "--h", "1/16", "--smoothers", "vanka"])
    assert r.returncode == 0 and len(_rows(r.stdout)) == 1 + 8
    r = _run(["paradiag", "--h", "1/16", "--tau", "1/16"])
    assert r.returncode == 0 and len(_rows(r.stdout)) == 1 + 16
    assert "all_converged=true" in r.stderr and "relative_residual=" in r.stderr
    r = _run(["paradiag", "--h", "1/16", "--tau", "1/16", "--smoother", "jacobi", "--max-iter", "1"])
    assert r.returncode == 2 and "did not converge" in r.stderr


@pytest.mark.gpu
def test_cli_csv_values_match_oracle(oracle):
    """CSV value parity: `solve`'s residual history and `sweep`'s per-shift iterations / rates equal the oracle's
    on the same inputs (the CLI's --seed stream, tools/pdmg.cpp:137-147), to 1e-10 / 1e-5 relative."""
    from oracle_lib import Cfg

    r = _run(["solve", "--h", "1/32", "--lambda-re", "5", "--lambda-im", "-7", "--seed", "77"])
    assert r.returncode == 0, r.stderr
    hist = np.array([float(ln.split(",")[1]) for ln in _rows(r.stdout)[1:]])
    b = oracle.random_complex(77, 31 * 31).reshape(31, 31)
    ref = oracle.solve(32, 5 - 7j, Cfg(cycle="W", nu1=1, nu2=0, coarsest_n=8, tol=1e-8), b)
    assert len(hist) == ref["iterations"] + 1
    assert np.max(np.abs(hist - ref["hist"]) / ref["hist"][0]) < 1e-10
    r = _run(["sweep", "--example", "backward-heat", "--h", "1/32", "--tau", "1/8", "--smoothers", "vanka",
              "--seed", "5"])
    assert r.returncode == 0, r.stderr
    rows = [ln.split(",") for ln in _rows(r.stdout)[1:]]
    lams = np.array([float(x[1]) + 1j * float(x[2]) for x in rows])
    np.testing.assert_allclose(lams, cli.qbv_eigenvalues(8, 1 / 8, 0.01), rtol=1e-13)
    b = oracle.random_complex(5, 31 * 31).reshape(1, 31, 31)
    ref = oracle.solve_batch(32, lams, Cfg(cycle="W", nu1=1, nu2=0, coarsest_n=8, tol=1e-8),
                             np.repeat(b, len(lams), axis=0), threads=8)
    assert [int(x[5]) for x in rows] == ref["iterations"].tolist()
    np.testing.assert_allclose([float(x[7]) for x in rows], ref["rates"], rtol=1e-5)


@pytest.mark.gpu
def test_cli_paradiag_qbv_rows_in_reference_order(oracle):
    """paradiag --scheme backward-heat: row k is the reference's eigenvalue k, (1 - gamma zeta^{-k}) / tau
    (paradiag.cpp:100), with that slot's cycle count; the condition estimate is finite and not ill-conditioned."""
    r = _run(["paradiag", "--scheme", "backward-heat", "--h", "1/16", "--tau", "1/8"])
    assert r.returncode == 0, r.stderr
    rows = [ln.split(",") for ln in _rows(r.stdout)[1:]]
    lams = np.array([float(x[1]) + 1j * float(x[2]) for x in rows])
    np.testing.assert_allclose(lams, cli.qbv_eigenvalues(8, 1 / 8, 0.01), rtol=1e-13)
    cond = float(r.stderr.split("cond_estimate=")[1].split()[0])
    assert math.isfinite(cond) and cond < 1e12 and "ill_conditioned=false" in r.stderr


@pytest.mark.gpu
def test_cli_lfa_table():
    """test_cli.cpp:143-151: lfa-table with two smoother rows; the Vanka row reproduces the README table
    (proj/README.md:108-112) at h = 1/256."""
    r = _run(["lfa-table", "--h", "1/32", "--tau", "1/32", "--samples", "16", "--nu-max", "2"])
    assert r.returncode == 0, r.stderr
    assert "smoother,omega_opt,mu,rho_nu1,rho_nu2" in r.stdout
    rows = _rows(r.stdout)[1:]
    assert len(rows) == 2 and rows[0].startswith("vanka,") and rows[1].startswith("jacobi,")
    r = _run(["lfa-table", "--smoothers", "vanka"])
    assert r.returncode == 0, r.stderr
    v = [float(x) for x in _rows(r.stdout)[1].split(",")[1:]]
    assert [round(x, 2) for x in v[:1]] == [0.96] and [round(x, 4) for x in v[1:]] == [0.28, 0.28, 0.1164, 0.0824, 0.0638]
