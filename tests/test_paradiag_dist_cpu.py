"""The multi-GPU ParaDIAG choreography (paper_2203_11154_b200/paradiag_dist.py) on CPU: world_size 2 over
gloo, with the local operators played by numpy (time DFT), the oracle (shifted solves) and a numpy
all-at-once residual.  The gathered result must equal the single-process oracle ParaDIAG."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

N_, NT, ALPHA = 16, 8, 0.01


class CpuOps:
    def __init__(self, n, nt, alpha, dt):
        import sys

        sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
        from oracle_lib import Cfg, Oracle

        self.o, self.cfg = Oracle(), Cfg()
        self.n, self.nt, self.alpha, self.dt = n, nt, alpha, dt
        self.sc = alpha ** (np.arange(nt) / nt)
        self.lams = self.o.circulant_shifts(alpha, nt, dt)

    @staticmethod
    def _c(x):
        return x.numpy().view(np.complex128)[..., 0]

    @staticmethod
    def _t(z):
        return torch.from_numpy(np.ascontiguousarray(z).astype(np.complex128)[..., None].view(np.float64).copy())

    def time_dft(self, x, step):
        z = self._c(x)
        if step == 1:
            return self._t(np.fft.ifft(self.sc[:, None] * z, axis=0))
        return self._t(np.fft.fft(z, axis=0) / self.sc[:, None])

    def solve(self, k0, k1, b):
        m = self.n - 1
        z = self._c(b).reshape(k1 - k0, m, m)
        r = self.o.solve_batch(self.n, self.lams[k0:k1], self.cfg, z, threads=1)
        return self._t(r["u"].reshape(k1 - k0, m * m)), r["iterations"].tolist()

    def residual(self, u_local, u_prev, f_local, t0):
        m = self.n - 1
        u = self._c(u_local).reshape(-1, m, m)
        up = self._c(u_prev).reshape(m, m)
        f = self._c(f_local).reshape(-1, m, m)
        rr = ff = 0.0
        for tl in range(u.shape[0]):
            au = self.o.apply_shifted_laplacian(self.n, 0.0, u[tl])
            prev = u[tl - 1] if tl > 0 else up
            wp = -self.alpha / self.dt if t0 + tl == 0 else -1 / self.dt
            r = f[tl] - (au + u[tl] / self.dt + wp * prev)
            rr += float(np.sum(np.abs(r) ** 2))
            ff += float(np.sum(np.abs(f[tl]) ** 2))
        return rr, ff


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2203_11154_b200.paradiag_dist import paradiag_step

    ops = CpuOps(N_, NT, ALPHA, 1.0 / NT)
    m = N_ - 1
    f = ops.o.random_complex(4, NT * m * m).reshape(NT, m * m)
    ntl = NT // world
    f_local = CpuOps._t(f[rank * ntl:(rank + 1) * ntl])
    u_local, iters, relres = paradiag_step(f_local, N_, NT, ALPHA, 1.0 / NT, ops)
    np.save(os.path.join(outdir, f"u{rank}.npy"), CpuOps._c(u_local))
    np.save(os.path.join(outdir, f"it{rank}.npy"), np.array(iters))
    np.save(os.path.join(outdir, f"rr{rank}.npy"), np.array([relres]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_distributed_paradiag_matches_single_process(tmp_path, oracle, world):
    mp.spawn(_worker, args=(world, _port(), str(tmp_path)), nprocs=world, join=True)
    m = N_ - 1
    u = np.concatenate([np.load(tmp_path / f"u{r}.npy") for r in range(world)]).reshape(NT, m, m)
    it = np.concatenate([np.load(tmp_path / f"it{r}.npy") for r in range(world)])
    f = oracle.random_complex(4, NT * m * m).reshape(NT, m, m)
    from oracle_lib import Cfg

    ref = oracle.paradiag(N_, NT, ALPHA, 1.0 / NT, Cfg(), f, threads=2)
    assert it.tolist() == ref["iterations"].tolist()
    assert np.linalg.norm(u - ref["u"]) <= 1e-12 * np.linalg.norm(ref["u"])
    for r in range(world):
        assert abs(float(np.load(tmp_path / f"rr{r}.npy")[0]) - ref["relres"]) <= 1e-6 * ref["relres"] + 1e-15
