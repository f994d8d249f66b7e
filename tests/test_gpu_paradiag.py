"""GPU ParaDIAG (alpha-circulant backward Euler) vs the oracle restatement (oracle/pdmg_oracle.c
orc_paradiag_circulant): identical per-slot cycle counts, solution within 1e-10 relative, and the
all-at-once residual at the multigrid tolerance."""
import numpy as np
import pytest
import torch

from oracle_lib import Cfg

pytestmark = pytest.mark.gpu

import paper_2203_11154_b200 as P  # noqa: E402
from paper_2203_11154_b200 import _native as N  # noqa: E402
from paper_2203_11154_b200.paradiag import ParadiagCirculant, heat_initial_rhs  # noqa: E402


def rel(a, b):
    return np.linalg.norm((a - b).ravel()) / np.linalg.norm(b.ravel())


@pytest.mark.parametrize("nt", [2, 6, 8, 32])
def test_time_dft_matches_numpy(nt):
    npts, alpha = 1000, 0.01
    rng = np.random.default_rng(nt)
    x = rng.standard_normal((nt, npts)) + 1j * rng.standard_normal((nt, npts))
    sc = alpha ** (np.arange(nt) / nt)
    dx = torch.from_numpy(x.view(np.float64)).cuda()
    dy = torch.empty_like(dx)
    assert N.lib().pdmg_time_dft(0, nt, npts, alpha, 1, dx.data_ptr(), dy.data_ptr(), None) == 0
    g = dy.cpu().numpy().view(np.complex128)
    np.testing.assert_allclose(g, np.fft.ifft(sc[:, None] * x, axis=0), rtol=0, atol=1e-13)
    assert N.lib().pdmg_time_dft(0, nt, npts, alpha, 3, dy.data_ptr(), dx.data_ptr(), None) == 0
    back = dx.cpu().numpy().view(np.complex128)
    np.testing.assert_allclose(back, x, rtol=0, atol=1e-12)


@pytest.mark.parametrize("n,nt", [(16, 8), (16, 6), (32, 16)])
def test_paradiag_matches_oracle(oracle, n, nt):
    m = n - 1
    alpha, dt = 0.01, 1.0 / nt
    f = oracle.random_complex(4, nt * m * m).reshape(nt, m, m)
    cfg = P.MultigridConfig(P.CycleKind.V, 1, 1, 4, 1e-10, 200, P.SmootherConfig.vanka())
    with ParadiagCirculant(n, nt, alpha, dt, cfg) as pd:
        u, reps, relres = pd.run(f)
    ref = oracle.paradiag(n, nt, alpha, dt, Cfg(), f, threads=8)
    assert [r.iterations for r in reps] == ref["iterations"].tolist()
    assert rel(u, ref["u"]) < 1e-10
    assert relres < 1e-9 and abs(relres - ref["relres"]) < 1e-10
    # the residual the GPU reports equals the oracle's evaluation of the GPU answer
    assert abs(oracle.all_at_once_residual_norm(n, nt, alpha, dt, u, f) /
               np.linalg.norm(f) - relres) < 1e-12


def test_config5_heat_step(oracle):
    """BASELINE config 5: 255x255 interior, 256 time steps, T=1, alpha=0.01, V(1,1), complex128."""
    n, nt = 256, 256
    dt, alpha = 1.0 / nt, 0.01
    f = heat_initial_rhs(n, nt, dt, seed=4)
    cfg = P.MultigridConfig(P.CycleKind.V, 1, 1, 4, 1e-10, 200, P.SmootherConfig.vanka())
    with ParadiagCirculant(n, nt, alpha, dt, cfg) as pd:
        u, reps, relres = pd.run(f)
    assert all(r.converged for r in reps)
    ref = oracle.paradiag(n, nt, alpha, dt, Cfg(), f, threads=16)
    assert [r.iterations for r in reps] == ref["iterations"].tolist()
    assert rel(u, ref["u"]) < 1e-10
    # each slot is solved to 1e-10 of its transformed rhs; alpha^(-t/nt) (up to 1/alpha) re-amplifies
    # the late slices on the way back, so the all-at-once residual sits near 1e-9 -- same as the oracle's
    assert relres < 1e-8 and abs(relres - ref["relres"]) <= 1e-3 * ref["relres"]


def test_qbv_tiny_matches_dense_kronecker(oracle):
    """test_paradiag.cpp:214-226 on the GPU: BackwardHeatQBV (alpha = -1/beta) vs the dense all-at-once solve."""
    td = P.TimeDiscretization(P.TimeSchemeKind.BackwardHeatQBV, 4, 0.25, 0.01)
    n, m, nt = 4, 3, td.dim()
    B = P.time_stepping_matrix(td)
    K = np.kron(B, np.eye(m * m)) + np.kron(np.eye(nt), oracle.dense_operator(n, 0.0))
    f = np.stack([oracle.random_complex(50 + i, m * m) for i in range(nt)]).reshape(nt, m, m)
    want = np.linalg.solve(K, f.ravel())
    cfg = P.MultigridConfig(coarsest_n=4)
    u, reps, relres = P.paradiag_solve(f, td, cfg)
    assert all(r.converged for r in reps)
    assert np.linalg.norm(u.ravel() - want) <= 1e-8 * np.linalg.norm(want)
    assert relres <= 1e-10


def test_qbv_matches_oracle(oracle):
    td = P.TimeDiscretization(P.TimeSchemeKind.BackwardHeatQBV, 8, 1.0 / 8, 0.01)
    n, m, nt = 32, 31, td.dim()
    f = oracle.random_complex(7, nt * m * m).reshape(nt, m, m)
    cfg = P.MultigridConfig(P.CycleKind.V, 1, 1, 4, 1e-10, 200, P.SmootherConfig.vanka())
    u, reps, relres = P.paradiag_solve(f, td, cfg)
    ref = oracle.paradiag(n, nt, td.circulant_alpha(), td.tau, Cfg(), f, threads=8)
    # paradiag_solve reports in the reference's eigenvalue order (paradiag.cpp:100): index k is circulant slot -k
    slots = P.paradiag.qbv_slot_of_reference_index(nt)
    assert [r.iterations for r in reps] == ref["iterations"][slots].tolist()
    lam_ref = P.diagonalize_qbv_closed_form(td).eigenvalues
    np.testing.assert_allclose(lam_ref, P.circulant_shifts(td.circulant_alpha(), nt, td.tau)[slots], rtol=1e-13)
    assert rel(u, ref["u"]) < 1e-10
    assert abs(relres - ref["relres"]) <= 1e-3 * ref["relres"] + 1e-14


def test_qbv_manufactured_run():
    """'manufactured space-time run converges with a small residual' (test_paradiag.cpp:230-250), QBV scheme,
    reference W(1,0) preset: relres <= 1e-6 and the manufactured field is recovered to 1e-5."""
    n = 16
    td = P.TimeDiscretization(P.TimeSchemeKind.BackwardHeatQBV, n, 1.0 / n, 0.01)
    ustar = P.manufactured_field(n, td.dim(), td.tau)
    f = P.all_at_once_apply(P.time_stepping_matrix(td), ustar)
    u, reps, relres = P.paradiag_solve(f, td, P.MultigridConfig())
    assert all(r.converged for r in reps)
    assert relres <= 1e-6
    err = max(np.linalg.norm(u[i] - ustar[i]) / np.linalg.norm(ustar[i]) for i in range(td.dim()))
    assert err <= 1e-5


def test_heat_bvm_tiny_matches_dense_kronecker(oracle):
    """'space-time solve matches a dense oracle on a tiny problem' (test_paradiag.cpp:198-212): HeatBVM,
    4 slices x 9 unknowns, general eigendecomposition + GPU GEMM time transforms."""
    td = P.TimeDiscretization(P.TimeSchemeKind.HeatBVM, 4, 0.25, 0.01)
    n, m, nt = 4, 3, td.dim()
    f = np.stack([oracle.random_complex(1 + i, m * m) for i in range(nt)]).reshape(nt, m, m)
    B = P.time_stepping_matrix(td)
    K = np.kron(B, np.eye(m * m)) + np.kron(np.eye(nt), oracle.dense_operator(n, 0.0))
    want = np.linalg.solve(K, f.ravel())
    u, reps, relres = P.paradiag_solve(f, td, P.MultigridConfig(coarsest_n=4))
    assert all(r.converged for r in reps)
    assert np.linalg.norm(u.ravel() - want) <= 1e-8 * np.linalg.norm(want)
    assert relres <= 1e-10


def test_heat_bvm_manufactured_run():
    """'manufactured space-time run converges with a small residual' (test_paradiag.cpp:230-250): HeatBVM,
    n = 16, tau = 1/16, reference W(1,0) preset: relres <= 1e-6, manufactured error <= 1e-5."""
    n = 16
    td = P.TimeDiscretization(P.TimeSchemeKind.HeatBVM, n, 1.0 / n, 0.01)
    ustar = P.manufactured_field(n, td.dim(), td.tau)
    f = P.all_at_once_apply(P.time_stepping_matrix(td), ustar)
    u, reps, relres = P.paradiag_solve(f, td, P.MultigridConfig())
    assert all(r.converged for r in reps)
    assert relres <= 1e-6
    err = max(np.linalg.norm(u[i] - ustar[i]) / np.linalg.norm(ustar[i]) for i in range(td.dim()))
    assert err <= 1e-5


@pytest.mark.parametrize("devices", [[0, 0], [0, 0, 0]])
def test_paradiag_device_list_matches_single(oracle, devices):
    """ParaDIAG with the time slices sharded over a device list (here shards sharing GPU 0, each with its own
    engine and stream): both time transforms gather their columns from every shard and scatter the rows to
    their owners inside the kernel; the result is bitwise the single-device one (the per-point transform
    arithmetic does not depend on the sharding) and relres agrees to summation order."""
    n, nt = 32, 10  # 10 slices over 3 shards: 4, 4, 2 (paradiag.cpp:222 chunking); not a power of two
    m = n - 1
    alpha, dt = 0.01, 1.0 / nt
    f = oracle.random_complex(9, nt * m * m).reshape(nt, m, m)
    cfg = P.MultigridConfig(P.CycleKind.V, 1, 1, 4, 1e-10, 200, P.SmootherConfig.vanka())
    with ParadiagCirculant(n, nt, alpha, dt, cfg) as pd:
        u1, reps1, rr1 = pd.run(f)
    with ParadiagCirculant(n, nt, alpha, dt, cfg, devices=devices) as pd:
        parts = pd.parts()
        u2, reps2, rr2 = pd.run(f)
    chunk = -(-nt // len(devices))
    assert parts[0] == (0, chunk, 0) and sum(p[1] for p in parts) == nt
    assert np.array_equal(u1, u2)
    assert [r.iterations for r in reps1] == [r.iterations for r in reps2]
    assert abs(rr1 - rr2) <= 1e-12 * rr1


def test_paradiag_shards_device_resident(oracle):
    """pdmg_paradiag_run_shards: per-shard device buffers."""
    n, nt = 32, 8
    m = n - 1
    f = oracle.random_complex(10, nt * m * m).reshape(nt, m, m)
    cfg = P.MultigridConfig(P.CycleKind.V, 1, 1, 4, 1e-10, 200, P.SmootherConfig.vanka())
    with ParadiagCirculant(n, nt, 0.01, 1.0 / nt, cfg) as pd:
        u1, _, rr1 = pd.run(f)
    with ParadiagCirculant(n, nt, 0.01, 1.0 / nt, cfg, devices=[0, 0]) as pd:
        d_f = [torch.from_numpy(np.ascontiguousarray(f[t0:t0 + c]).view(np.float64)).cuda() for t0, c, _ in pd.parts()]
        d_u = [torch.empty_like(x) for x in d_f]
        reps, rr2 = pd.run_shards([x.data_ptr() for x in d_f], [x.data_ptr() for x in d_u], want_reports=True)
        torch.cuda.synchronize()
        u2 = np.concatenate([x.cpu().numpy().view(np.complex128).reshape(-1, m, m) for x in d_u])
    assert np.array_equal(u1, u2) and abs(rr1 - rr2) <= 1e-12 * rr1
    assert all(r.converged for r in reps)


@pytest.mark.parametrize("nt,npts", [(1, 7), (5, 1000), (33, 4099), (64, 20000)])
def test_time_transform_kernel_matches_numpy(nt, npts):
    """The hand-written complex fp64 GEMM over the time index (k_time_gemm; kron_time_apply, paradiag.cpp:129-133)
    against numpy, ragged in both the time and the point dimensions."""
    rng = np.random.default_rng(nt)
    M = rng.standard_normal((nt, nt)) + 1j * rng.standard_normal((nt, nt))
    x = rng.standard_normal((nt, npts)) + 1j * rng.standard_normal((nt, npts))
    dx = torch.from_numpy(x.view(np.float64)).cuda()
    dy = torch.empty_like(dx)
    Mc = np.ascontiguousarray(M)
    assert N.lib().pdmg_time_transform(0, nt, npts, Mc.ctypes.data, dx.data_ptr(), dy.data_ptr(), None) == 0
    y = dy.cpu().numpy().view(np.complex128)
    np.testing.assert_allclose(y, M @ x, rtol=0, atol=1e-12 * max(1.0, np.abs(M @ x).max()))


@pytest.mark.parametrize("devices", [None, [0, 0]])
def test_heat_bvm_general_scheme_matches_oracle_solves(oracle, devices):
    """HeatBVM through the general scheme (hand-written time GEMMs), one device and sharded: every slot's
    shifted solve matches the oracle's batched solve of the same transformed right-hand side, and the
    all-at-once residual is at the multigrid tolerance."""
    n = 32
    td = P.TimeDiscretization(P.TimeSchemeKind.HeatBVM, 8, 1.0 / 8, 0.01)
    m, nt = n - 1, td.dim()
    f = oracle.random_complex(12, nt * m * m).reshape(nt, m, m)
    cfg = P.MultigridConfig(P.CycleKind.V, 1, 1, 4, 1e-10, 200, P.SmootherConfig.vanka())
    B = P.time_stepping_matrix(td)
    dg = P.diagonalize_time_matrix(B)
    with P.ParadiagGeneral(n, B, dg, cfg, devices=devices) as pd:
        u, reps, relres = pd.run(f)
    g = (dg.Vinv @ f.reshape(nt, -1)).reshape(nt, m, m)
    ref = oracle.solve_batch(n, dg.eigenvalues, Cfg(), g, threads=8)
    assert [r.iterations for r in reps] == ref["iterations"].tolist()
    u_ref = (dg.V @ ref["u"].reshape(nt, -1)).reshape(nt, m, m)
    assert rel(u, u_ref) < 1e-10
    assert relres < 1e-8


def test_paradiag_ipc_ranks_match_single_process():
    """Rank mode (one process per GPU): two torchrun ranks -- both on GPU 0 here, each owning half the time slices
    in its own process -- exchange CUDA IPC handles and run the fused gather/scatter transforms across the two
    processes (tests/ipc_paradiag_worker.py); the result is bitwise the single-process solver's."""
    import os
    import socket
    import subprocess
    import sys

    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port),
                        os.path.join(root, "tests", "ipc_paradiag_worker.py")], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "ipc paradiag ok" in r.stdout
