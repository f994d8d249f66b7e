"""Worker of tests/test_gpu_paradiag.py::test_paradiag_ipc_ranks_match_single_process (torchrun, 2 ranks).

Both ranks run on GPU 0 (this pool's boxes have one B200): each owns half the time slices in its own process,
the ranks open each other's slice buffers over CUDA IPC, and the fused transform kernels gather / scatter across
the two processes.  The kernels never wait on each other: the phases are separated by process barriers.  Rank 0
checks the result against the single-process solver: bitwise u, the same cycle counts, relres to rounding."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2203_11154_b200 as P  # noqa: E402
from paper_2203_11154_b200.paradiag import ParadiagCirculant  # noqa: E402
from paper_2203_11154_b200.paradiag_dist import IpcParadiag  # noqa: E402


class DevView:
    """A device buffer owned by libpdmg_b200 as a torch tensor (zero-copy, __cuda_array_interface__)."""

    def __init__(self, ptr, count):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": "<f8", "data": (ptr, False), "version": 3}


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    n, nt, alpha, dt = 32, 10, 0.01, 0.1
    m = n - 1
    cfg = P.MultigridConfig(P.CycleKind.V, 1, 1, 4, 1e-10, 200, P.SmootherConfig.vanka())
    f = P.random_rhs(n, 9, count=nt)
    pd = IpcParadiag(n, nt, alpha, dt, cfg, device=0)
    fv = torch.as_tensor(DevView(pd.f_ptr, pd.ntl * m * m * 2), device="cuda:0")
    fv.copy_(torch.from_numpy(np.ascontiguousarray(f[pd.t0:pd.t0 + pd.ntl]).view(np.float64).ravel()))
    torch.cuda.synchronize()
    iters, relres = pd.step()
    uv = torch.as_tensor(DevView(pd.u_ptr, pd.ntl * m * m * 2), device="cuda:0").cpu().numpy()
    u_local = uv.view(np.complex128).reshape(pd.ntl, m, m)
    parts = [None] * world
    dist.all_gather_object(parts, (pd.t0, u_local, iters, relres))
    pd.close()
    if rank == 0:
        u = np.concatenate([p[1] for p in sorted(parts, key=lambda p: p[0])])
        it = sum((p[2] for p in sorted(parts, key=lambda p: p[0])), [])
        with ParadiagCirculant(n, nt, alpha, dt, cfg) as ref:
            u1, reps1, rr1 = ref.run(f)
        assert np.array_equal(u, u1), float(np.abs(u - u1).max())
        assert it == [r.iterations for r in reps1], (it, [r.iterations for r in reps1])
        assert abs(relres - rr1) <= 1e-12 * rr1, (relres, rr1)
        print("ipc paradiag ok", it, relres, flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
