"""pdmg-b200 command-line driver: `solve`, `sweep`, `paradiag` on the GPU backend.

Mirrors the reference CLI (proj/tools/pdmg.cpp:226-516) -- same subcommands, options, defaults, CSV columns,
'#'-manifest block (proj/src/runio.cpp:39-82) and exit codes (0 ok, 1 usage/configuration error, 2 numerical
failure; pdmg.cpp:27-29, 520-554).  `lfa-table` is out of scope (offline Fourier analysis).
Differences: `sweep` batches all shifts of a smoother into one GPU solve; `paradiag --threads` is accepted and
ignored (the shifted solves run batched on the GPU); HeatBVM eigenvalues come from LAPACK (numpy) rather than
Eigen, so their order -- and hence `--shift-index` for `--scheme heat-bvm` -- may differ.

    python -m paper_2203_11154_b200.cli solve --h 1/64 --lambda-re 8.959 --lambda-im -15.395 --cycle v \\
        --nu1 1 --nu2 1 --h0 1/4 --tol 1e-10 --seed 0
"""
from __future__ import annotations

import argparse
import math
import sys
import time

import numpy as np

from . import multigrid as M
from . import paradiag as PD

VERSION = "0.1.0+b200"
EXIT_OK, EXIT_USAGE, EXIT_NUMERICAL = 0, 1, 2


# ---- runio (proj/src/runio.cpp) restated --------------------------------------------------------------
def parse_real(text: str) -> float:
    try:
        return float(text)
    except ValueError:
        raise M.ConfigError(f"could not parse '{text}' as a number")


def parse_reciprocal(text: str) -> int:
    """runio.cpp:19-37: 'p/q' or a decimal that is the reciprocal of an integer, in (0, 1/2]."""
    if "/" in text:
        num, den = text.split("/", 1)
        num, den = parse_real(num), parse_real(den)
        if den == 0.0:
            raise M.ConfigError(f"division by zero in '{text}'")
        value = num / den
    else:
        value = parse_real(text)
    if not (value > 0.0) or not (value <= 0.5):
        raise M.ConfigError(f"'{text}' is out of range: need a value in (0, 1/2]")
    inv = 1.0 / value
    r = round(inv)
    if abs(inv - r) > 1e-9 * r:
        raise M.ConfigError(f"'{text}' is not the reciprocal of an integer")
    return int(r)


def format_sig(v: float) -> str:
    return "%.15g" % v


def fnv1a_hex(data: str) -> str:
    h = 14695981039346656037
    for c in data.encode():
        h ^= c
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return "%016x" % h


class RunManifest:
    def __init__(self, command: str):
        self.command, self.parameters, self.version = command, [], VERSION

    def add(self, k: str, v: str):
        self.parameters.append((k, v))

    def canonical(self) -> str:
        return f"command={self.command};version={self.version}" + "".join(f";{k}={v}" for k, v in self.parameters)

    def write_comments(self, os):
        os.write(f"# pdmg {self.command} v{self.version}\n# manifest-hash: {fnv1a_hex(self.canonical())}\n")
        for k, v in self.parameters:
            os.write(f"# {k} = {v}\n")


class CsvWriter:
    def __init__(self, os, manifest: RunManifest, columns):
        self.os, self.n = os, len(columns)
        manifest.write_comments(os)
        os.write(",".join(columns) + "\n")

    def row(self, cells):
        if len(cells) != self.n:
            raise M.ConfigError(f"CsvWriter: row has {len(cells)} cells, expected {self.n}")
        self.os.write(",".join(cells) + "\n")


def bool_str(v: bool) -> str:
    return "true" if v else "false"


# ---- shared options (pdmg.cpp:62-102) ------------------------------------------------------------------
def add_cycle_opts(p):
    p.add_argument("--cycle", default="w", choices=["v", "w"])
    p.add_argument("--nu1", type=int, default=1)
    p.add_argument("--nu2", type=int, default=0)
    p.add_argument("--h0", default="1/8")
    p.add_argument("--tol", type=float, default=1e-8)
    p.add_argument("--max-iter", type=int, default=200)
    p.add_argument("-o", "--out", default="-")
    p.add_argument("--device", type=int, default=0, help="CUDA device (B200 extension)")


def make_cfg(a, kind: M.SmootherKind, omega: float) -> M.MultigridConfig:
    sm = M.SmootherConfig(kind, omega)
    return M.MultigridConfig(M.CycleKind.V if a.cycle == "v" else M.CycleKind.W, a.nu1, a.nu2,
                             parse_reciprocal(a.h0), a.tol, a.max_iter, sm)


def describe_cycle(a, m: RunManifest):
    m.add("cycle", a.cycle)
    m.add("nu1", str(a.nu1))
    m.add("nu2", str(a.nu2))
    m.add("h0", "1/" + str(parse_reciprocal(a.h0)))
    m.add("tol", format_sig(a.tol))
    m.add("max_iter", str(a.max_iter))


def parse_smoother(name: str) -> M.SmootherKind:
    if name == "vanka":
        return M.SmootherKind.Vanka
    if name == "jacobi":
        return M.SmootherKind.Jacobi
    raise M.ConfigError(f"unknown smoother '{name}' (expected vanka or jacobi)")


def preset_omega(k: M.SmootherKind) -> float:
    return 24.0 / 25.0 if k == M.SmootherKind.Vanka else 4.0 / 5.0


def open_out(path):
    return sys.stdout if path == "-" else open(path, "w")


def qbv_eigenvalues(n: int, tau: float, beta: float) -> np.ndarray:
    """diagonalize_qbv_closed_form eigenvalue order (paradiag.cpp:84-108): (1 - gamma zeta^{-k}) / tau."""
    return PD.diagonalize_qbv_closed_form(PD.TimeDiscretization(PD.TimeSchemeKind.BackwardHeatQBV, n, tau,
                                                                beta)).eigenvalues


def scheme_shifts(scheme: str, n: int, beta: float) -> np.ndarray:
    if scheme in ("heat-bvm", "heat"):
        td = PD.TimeDiscretization(PD.TimeSchemeKind.HeatBVM, n, 1.0 / n, beta)
        return PD.diagonalize_time_matrix(PD.time_stepping_matrix(td)).eigenvalues
    return qbv_eigenvalues(n, 1.0 / n, beta)


# ---- subcommands ---------------------------------------------------------------------------------------
def cmd_solve(a) -> int:
    N = parse_reciprocal(a.h)
    grid = M.Grid2D(N)
    if a.scheme is None:
        lam = complex(a.lambda_re or 0.0, a.lambda_im)
    else:
        if a.lambda_re is not None or a.lambda_im != 0.0:
            raise M.ConfigError("--lambda-re/--lambda-im and --scheme are mutually exclusive")
        fam = (PD.helmholtz_shifts(grid.h) if a.scheme == "helmholtz"
               else scheme_shifts(a.scheme, parse_reciprocal(a.tau or a.h), a.beta))
        if not 1 <= a.shift_index <= len(fam):
            raise M.ConfigError(f"--shift-index out of range (family has {len(fam)} shifts)")
        lam = complex(fam[a.shift_index - 1])
    kind = parse_smoother(a.smoother)
    w = a.omega if a.omega > 0.0 else preset_omega(kind)
    cfg = make_cfg(a, kind, w)
    if a.rhs == "manufactured":
        ustar = PD.manufactured_field(grid, 1, 0.0)[0]
        z = np.pad(ustar, 1)
        b = (4 * z[1:-1, 1:-1] - z[:-2, 1:-1] - z[2:, 1:-1] - z[1:-1, :-2] - z[1:-1, 2:]) * N * N + lam * ustar
    else:
        b = M.random_rhs(grid, a.seed)
    u, rep = M.multigrid_solve(b, M.Shift(lam), cfg, a.device)
    m = RunManifest("solve")
    m.add("h", f"1/{N}")
    m.add("lambda_re", format_sig(lam.real))
    m.add("lambda_im", format_sig(lam.imag))
    m.add("smoother", a.smoother)
    m.add("omega", format_sig(w))
    m.add("rhs", a.rhs)
    if a.rhs == "random":
        m.add("seed", str(a.seed))
    describe_cycle(a, m)
    os = open_out(a.out)
    csv = CsvWriter(os, m, ["iter", "residual"])
    for k, r in enumerate(rep.residual_history):
        csv.row([str(k), format_sig(r)])
    if os is not sys.stdout:
        os.close()
    sys.stderr.write(f"solve: converged={bool_str(rep.converged)} iterations={rep.iterations} "
                     f"rate={format_sig(rep.rate)} seconds={format_sig(rep.seconds)}\n")
    return EXIT_OK


def cmd_lfa_table(a) -> int:
    """lfa-table (pdmg.cpp:153-220): optimized damping, smoothing factor and two-grid factors rho(1..nu_max) per
    smoother for the first eigenvalue shift of the time scheme, from the GPU LFA kernels."""
    from . import lfa as LFA

    N_ = parse_reciprocal(a.h)
    n = parse_reciprocal(a.tau or a.h)
    shift = complex(scheme_shifts(a.scheme, n, a.beta)[0])
    if a.nu_max < 1:
        raise M.ConfigError("--nu-max must be positive")
    kinds = [parse_smoother(s) for s in a.smoothers.split(",") if s]
    if not kinds:
        raise M.ConfigError("--smoothers: empty list")
    cfg = LFA.LFAConfig(a.samples, 1e-8)
    cfg.validate()
    m = RunManifest("lfa-table")
    m.add("h", f"1/{N_}")
    m.add("tau", f"1/{n}")
    m.add("scheme", a.scheme)
    if a.scheme == "backward-heat":
        m.add("beta", format_sig(a.beta))
    m.add("lambda_re", format_sig(shift.real))
    m.add("lambda_im", format_sig(shift.imag))
    m.add("samples", str(a.samples))
    m.add("nu_max", str(a.nu_max))
    os = open_out(a.out)
    csv = CsvWriter(os, m, ["smoother", "omega_opt", "mu"] + [f"rho_nu{nu}" for nu in range(1, a.nu_max + 1)])
    for kind in kinds:
        model = LFA.TwoGridModel(shift, 1.0 / N_, kind, cfg, a.device)
        opt = LFA.optimize_omega(model, LFA.OmegaObjective.TwoGridRho, 1)
        name = "vanka" if kind == M.SmootherKind.Vanka else "jacobi"
        csv.row([name, format_sig(opt.omega), format_sig(model.smoothing(opt.omega).mu)]
                + [format_sig(model.rho(opt.omega, nu)) for nu in range(1, a.nu_max + 1)])
        sys.stderr.write(f"lfa-table: {name} omega_opt={format_sig(opt.omega)} rho1={format_sig(opt.value)}\n")
    if os is not sys.stdout:
        os.close()
    return EXIT_OK


def cmd_sweep(a) -> int:
    N = parse_reciprocal(a.h)
    grid = M.Grid2D(N)
    if a.example == "helmholtz":
        tau_desc, lams = "n/a", PD.helmholtz_shifts(grid.h)
    else:
        n = parse_reciprocal(a.tau or a.h)
        tau_desc, lams = f"1/{n}", scheme_shifts(a.example, n, a.beta)
    kinds = [parse_smoother(s) for s in a.smoothers.split(",") if s]
    if not kinds:
        raise M.ConfigError("--smoothers: empty list")
    b = M.random_rhs(grid, a.seed)
    m = RunManifest("sweep")
    m.add("example", a.example)
    m.add("h", f"1/{N}")
    m.add("tau", tau_desc)
    if a.example == "backward-heat":
        m.add("beta", format_sig(a.beta))
    m.add("smoothers", a.smoothers)
    m.add("omega_vanka", format_sig(a.omega_vanka))
    m.add("omega_jacobi", format_sig(a.omega_jacobi))
    m.add("seed", str(a.seed))
    describe_cycle(a, m)
    os = open_out(a.out)
    csv = CsvWriter(os, m, ["shift_index", "lambda_re", "lambda_im", "smoother", "omega", "iterations", "converged",
                            "rate"])
    bad = 0
    for kind in kinds:
        w = a.omega_vanka if kind == M.SmootherKind.Vanka else a.omega_jacobi
        cfg = make_cfg(a, kind, w)
        # all shifts of the family in one batched GPU solve (pdmg.cpp:406-417 loops multigrid_solve)
        with M.BatchedMultigridHierarchy(grid, list(lams), cfg, a.device) as H:
            _, reps = H.solve(np.broadcast_to(b, (len(lams),) + b.shape))
        for j, (lam, rep) in enumerate(zip(lams, reps)):
            bad += not rep.converged
            idx = j + 1 if a.example == "helmholtz" else j
            csv.row([str(idx), format_sig(lam.real), format_sig(lam.imag), "vanka" if kind == 0 else "jacobi",
                     format_sig(w), str(rep.iterations), bool_str(rep.converged), format_sig(rep.rate)])
    if os is not sys.stdout:
        os.close()
    sys.stderr.write(f"sweep: {len(lams)} shifts x {len(kinds)} smoothers, {bad} non-converged\n")
    return EXIT_OK


def cmd_paradiag(a) -> int:
    t0 = time.perf_counter()
    N = parse_reciprocal(a.h)
    grid = M.Grid2D(N)
    n = parse_reciprocal(a.tau or a.h)
    kind_t = PD.TimeSchemeKind.HeatBVM if a.scheme == "heat-bvm" else PD.TimeSchemeKind.BackwardHeatQBV
    td = PD.TimeDiscretization(kind_t, n, 1.0 / n, a.beta)
    kind = parse_smoother(a.smoother)
    w = a.omega if a.omega > 0.0 else preset_omega(kind)
    cfg = make_cfg(a, kind, w)
    ustar = PD.manufactured_field(grid, td.dim(), td.tau)
    f = PD.all_at_once_apply(PD.time_stepping_matrix(td), ustar)
    u, reps, relres = PD.paradiag_solve(f, td, cfg, a.device)
    rel_err = math.sqrt(float(np.sum(np.abs(u - ustar) ** 2)) / float(np.sum(np.abs(ustar) ** 2)))
    if kind_t == PD.TimeSchemeKind.HeatBVM:
        dg = PD.diagonalize_time_matrix(PD.time_stepping_matrix(td))
        lams, cond = dg.eigenvalues, dg.cond_estimate
    else:  # reference eigenvalue order (paradiag_solve already reports in it)
        dg = PD.diagonalize_qbv_closed_form(td)
        lams, cond = dg.eigenvalues, dg.cond_estimate
    m = RunManifest("paradiag")
    m.add("scheme", a.scheme)
    m.add("h", f"1/{N}")
    m.add("tau", f"1/{n}")
    if kind_t == PD.TimeSchemeKind.BackwardHeatQBV:
        m.add("beta", format_sig(a.beta))
    m.add("smoother", a.smoother)
    m.add("omega", format_sig(w))
    m.add("threads", str(a.threads))
    describe_cycle(a, m)
    os = open_out(a.out)
    csv = CsvWriter(os, m, ["shift_index", "lambda_re", "lambda_im", "iterations", "converged", "rate"])
    for j, rep in enumerate(reps):
        csv.row([str(j), format_sig(lams[j].real), format_sig(lams[j].imag), str(rep.iterations),
                 bool_str(rep.converged), format_sig(rep.rate)])
    if os is not sys.stdout:
        os.close()
    allc = all(r.converged for r in reps)
    sys.stderr.write(f"paradiag: relative_residual={format_sig(relres)} manufactured_error={format_sig(rel_err)} "
                     f"cond_estimate={format_sig(cond)} ill_conditioned={bool_str(not cond <= 1e12)} "
                     f"all_converged={bool_str(allc)} seconds={format_sig(time.perf_counter() - t0)}\n")
    if not allc:
        sys.stderr.write("paradiag: at least one shifted solve did not converge\n")
        return EXIT_NUMERICAL
    return EXIT_OK


def build_parser():
    ap = argparse.ArgumentParser(prog="pdmg-b200", description="B200 shifted-Laplacian multigrid driver")
    ap.add_argument("--version", action="version", version="pdmg " + VERSION)  # pdmg.cpp:523
    sub = ap.add_subparsers(dest="cmd", required=True)
    s = sub.add_parser("solve", help="Run one shifted multigrid solve and dump residual history")
    s.add_argument("--h", required=True)
    s.add_argument("--lambda-re", type=float, default=None)
    s.add_argument("--lambda-im", type=float, default=0.0)
    s.add_argument("--scheme", choices=["heat-bvm", "backward-heat", "helmholtz"])
    s.add_argument("--tau")
    s.add_argument("--beta", type=float, default=0.01)
    s.add_argument("--shift-index", type=int, default=1)
    s.add_argument("--smoother", default="vanka", choices=["vanka", "jacobi"])
    s.add_argument("--omega", type=float, default=0.0)
    s.add_argument("--rhs", default="random", choices=["random", "manufactured"])
    s.add_argument("--seed", type=int, default=1234)
    add_cycle_opts(s)
    s.set_defaults(fn=cmd_solve)
    t = sub.add_parser("lfa-table", help="Predicted smoothing/two-grid factors with optimized damping")
    t.add_argument("--h", default="1/256")
    t.add_argument("--tau")
    t.add_argument("--scheme", default="heat-bvm", choices=["heat-bvm", "backward-heat"])
    t.add_argument("--beta", type=float, default=0.01)
    t.add_argument("--smoothers", default="vanka,jacobi")
    t.add_argument("--nu-max", type=int, default=4)
    t.add_argument("--samples", type=int, default=64)
    t.add_argument("-o", "--out", default="-")
    t.add_argument("--device", type=int, default=0, help="CUDA device (B200 extension)")
    t.set_defaults(fn=cmd_lfa_table)
    w = sub.add_parser("sweep", help="Solve across a family of shifts and tabulate iterations/rates")
    w.add_argument("--example", required=True, choices=["heat", "backward-heat", "helmholtz"])
    w.add_argument("--h", required=True)
    w.add_argument("--tau")
    w.add_argument("--beta", type=float, default=0.01)
    w.add_argument("--smoothers", default="vanka,jacobi")
    w.add_argument("--omega-vanka", type=float, default=24.0 / 25.0)
    w.add_argument("--omega-jacobi", type=float, default=4.0 / 5.0)
    w.add_argument("--seed", type=int, default=1234)
    add_cycle_opts(w)
    w.set_defaults(fn=cmd_sweep)
    p = sub.add_parser("paradiag", help="Diagonalization-based space-time solve with a manufactured rhs")
    p.add_argument("--scheme", default="heat-bvm", choices=["heat-bvm", "backward-heat"])
    p.add_argument("--h", required=True)
    p.add_argument("--tau")
    p.add_argument("--beta", type=float, default=0.01)
    p.add_argument("--smoother", default="vanka", choices=["vanka", "jacobi"])
    p.add_argument("--omega", type=float, default=0.0)
    p.add_argument("--threads", type=int, default=1)
    add_cycle_opts(p)
    p.set_defaults(fn=cmd_paradiag)
    return ap


def main(argv=None) -> int:
    ap = build_parser()
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:  # argparse usage errors -> exit 1 like CLI11 (pdmg.cpp:535-541)
        return EXIT_USAGE if e.code else EXIT_OK
    try:
        if getattr(a, "threads", 1) < 1:
            raise M.ConfigError("--threads must be positive")
        return a.fn(a)
    except M.ConfigError as e:
        sys.stderr.write(f"error: {e}\n")
        return EXIT_USAGE
    except M.SingularOperatorError as e:
        sys.stderr.write(f"numerical error: {e}\n")
        return EXIT_NUMERICAL
    except M.DeviceError as e:
        sys.stderr.write(f"device error: {e}\n")
        return EXIT_NUMERICAL


if __name__ == "__main__":
    sys.exit(main())
