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
