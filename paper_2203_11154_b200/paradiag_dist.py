"""Multi-GPU ParaDIAG step (BASELINE config 5 on 1/2/4/8 GPUs), one process per GPU.

Two transports:
  * `IpcParadiag` (default): every rank owns its time slices in libpdmg_b200 (pdmg_paradiag_create_rank); the
    ranks exchange CUDA IPC handles of their slice buffers once, and the time-transform kernels gather each
    spatial point's time column from every rank and scatter the results to their owners through NVLink peer
    memory -- the all-to-all is inside the transform (the same kernels as the single-process device list).
  * `paradiag_step` + `GpuOps`: NCCL all-to-all transposes around the alpha-scaled time DFT (below).

Data movement; P = world size, nt divisible by P, points padded to P * pl:
    f  [t-shard][points]  --a2a-->  [t][point-shard]  --DFT step 1-->  [k][point-shard]
       --a2a-->  [k-shard][points]  --batched MG solve of the rank's lambda_k-->  w [k-shard][points]
       --a2a-->  [k][point-shard]  --DFT step 3-->  [t][point-shard]  --a2a-->  u [t-shard][points]
    relres: each rank needs u_{t0-1} (rank 0: u_{nt-1}) -> one ring send/recv; ||r||^2, ||f||^2 all-reduced.

The local operators are pluggable so the same choreography runs on GPUs (libpdmg_b200 kernels, NCCL)
and in the CPU tests (oracle + numpy, gloo).  Reference: paradiag_solve (proj/src/paradiag.cpp:185-248),
whose only parallelism is a std::thread pool over shifts (paradiag.cpp:217-236).
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def _a2a(x: torch.Tensor, world: int) -> torch.Tensor:
    """all_to_all over the leading (destination-rank) dimension of a contiguous float64 tensor."""
    out = torch.empty_like(x)
    dist.all_to_all_single(out, x.contiguous())
    return out


def paradiag_step(f_local: torch.Tensor, n: int, nt: int, alpha: float, dt: float, ops) -> tuple:
    """f_local: [ntl, m*m, 2] float64 (complex as pairs) on this rank's device; returns (u_local, iters, relres).

    ops must provide time_dft(x[nt, pl, 2], step) -> same shape; solve(k0, k1, b[kl, m*m, 2]) -> (w, iters);
    residual(u_local, u_prev, f_local, t0) -> (||r||^2, ||f||^2)."""
    world, rank = dist.get_world_size(), dist.get_rank()
    if nt % world:
        raise ValueError(f"paradiag_step: nt = {nt} must be divisible by the number of ranks {world}")
    ntl = nt // world
    npts = (n - 1) ** 2
    pl = -(-npts // world)
    pad = pl * world - npts
    t0 = rank * ntl
    dev = f_local.device

    def to_point_shards(x):  # [ntl, npts, 2] -> [ntl, world*pl, 2] -> [world, ntl, pl, 2]
        if pad:
            x = torch.cat([x, torch.zeros(x.shape[0], pad, 2, dtype=x.dtype, device=dev)], dim=1)
        return x.view(x.shape[0], world, pl, 2).transpose(0, 1).contiguous()

    def from_point_shards(y):  # [world(src), ntl, pl, 2] -> [ntl, npts, 2]
        return y.transpose(0, 1).reshape(y.shape[1], world * pl, 2)[:, :npts].contiguous()

    # step 1: f [t-shard] -> [t][point-shard] -> DFT -> [k][point-shard] -> [k-shard][points]
    x = _a2a(to_point_shards(f_local), world).view(nt, pl, 2)
    g_pts = ops.time_dft(x, 1)  # [nt(k), pl, 2]
    g = from_point_shards(_a2a(g_pts.view(world, ntl, pl, 2), world))
    # step 2: this rank's shifts lambda_k, k in [t0, t0+ntl)
    w, iters = ops.solve(t0, t0 + ntl, g)
    # step 3: w [k-shard][points] -> [k][point-shard] -> DFT back -> [t][point-shard] -> [t-shard][points]
    y = _a2a(to_point_shards(w), world).view(nt, pl, 2)
    u_pts = ops.time_dft(y, 3)
    u_local = from_point_shards(_a2a(u_pts.view(world, ntl, pl, 2), world))
    # all-at-once residual: ring exchange of the boundary slice u_{t0-1}
    u_prev = torch.empty(npts, 2, dtype=u_local.dtype, device=dev)
    send = u_local[ntl - 1].contiguous()
    reqs = [dist.isend(send, (rank + 1) % world), dist.irecv(u_prev, (rank - 1) % world)]
    for r in reqs:
        r.wait()
    rr, ff = ops.residual(u_local, u_prev, f_local, t0)
    sums = torch.tensor([rr, ff], dtype=torch.float64, device=dev)
    dist.all_reduce(sums)
    relres = float(torch.sqrt(sums[0]) / torch.sqrt(sums[1])) if float(sums[1]) > 0 else float(torch.sqrt(sums[0]))
    return u_local, iters, relres


class GpuOps:
    """Local operators on this rank's GPU through libpdmg_b200 (kernels run on torch's current stream)."""

    def __init__(self, n: int, nt: int, alpha: float, dt: float, cfg, device: int):
        from .multigrid import BatchedMultigridHierarchy, Grid2D, circulant_shifts

        self.n, self.nt, self.alpha, self.dt, self.device = n, nt, alpha, dt, device
        self.lams = circulant_shifts(alpha, nt, dt)
        self.cfg = cfg
        self._H = {}
        self._mk = lambda k0, k1: BatchedMultigridHierarchy(Grid2D(n), self.lams[k0:k1], cfg, device)

    def _stream(self):
        return torch.cuda.current_stream(self.device).cuda_stream

    def time_dft(self, x: torch.Tensor, step: int) -> torch.Tensor:
        from . import _native as N
        from .multigrid import _check

        y = torch.empty_like(x)
        _check(N.lib().pdmg_time_dft(self.device, self.nt, x.shape[1], self.alpha, step, x.data_ptr(), y.data_ptr(),
                                     self._stream()))
        return y

    def solve(self, k0: int, k1: int, b: torch.Tensor):
        key = (k0, k1)
        if key not in self._H:
            self._H[key] = self._mk(k0, k1)
        H = self._H[key]
        torch.cuda.current_stream(self.device).synchronize()
        w = torch.empty_like(b)
        reps = H.solve_device(b.data_ptr(), w.data_ptr())
        return w, [r.iterations for r in reps]

    def residual(self, u_local, u_prev, f_local, t0):
        import ctypes as C

        from . import _native as N
        from .multigrid import _check

        sums = (C.c_double * 2)()
        _check(N.lib().pdmg_aao_residual(self.device, self.n, u_local.shape[0], t0, self.alpha, self.dt,
                                         u_local.data_ptr(), u_prev.data_ptr(), f_local.data_ptr(), sums,
                                         self._stream()))
        return sums[0], sums[1]


class IpcParadiag:
    """One rank's share of a ParaDIAG solver whose time slices are sharded over the ranks of the default process
    group; peers' slice buffers are opened over CUDA IPC (pdmg_paradiag_create_rank / _ipc_handles / _open_peers).
    `step()` runs the four phases with a process barrier between them and returns (iterations of this rank's
    slots, relres)."""

    def __init__(self, n: int, nt: int, alpha: float, dt: float, cfg, device: int):
        import ctypes as C

        from . import _native as N
        from .multigrid import _check

        self.N, self.C, self._check = N, C, _check
        self.world, self.rank = dist.get_world_size(), dist.get_rank()
        self.n, self.nt, self.cfg = n, nt, cfg
        h = C.c_void_p()
        c = cfg._c()
        _check(N.lib().pdmg_paradiag_create_rank(n, nt, alpha, dt, C.byref(c), self.rank, self.world, device,
                                                 C.byref(h)))
        self._h = h
        mine = (C.c_char * 256)()
        _check(N.lib().pdmg_paradiag_ipc_handles(h, mine))
        allh = [None] * self.world
        dist.all_gather_object(allh, bytes(mine))
        buf = (C.c_char * (256 * self.world)).from_buffer_copy(b"".join(allh))
        _check(N.lib().pdmg_paradiag_open_peers(h, buf))
        self.chunk = -(-nt // self.world)
        self.t0 = self.rank * self.chunk
        self.ntl = min(nt, self.t0 + self.chunk) - self.t0
        self.f_ptr = N.lib().pdmg_paradiag_rank_buffer(h, 0)
        self.u_ptr = N.lib().pdmg_paradiag_rank_buffer(h, 3)
        dist.barrier()

    @property
    def solver_handle(self):
        return self.N.lib().pdmg_paradiag_solver(self._h)

    def step(self, want_iterations: bool = True):
        N, C, _check = self.N, self.C, self._check
        H = self.cfg.max_iter + 1
        it = np.zeros(self.nt, np.int32)
        rep = N.SolveReport(it.ctypes.data, None, None, None, 0.0) if want_iterations else None
        sums = (C.c_double * 2)()
        dist.barrier()  # every rank's f slices are in place
        for k in (1, 2, 3, 4):
            _check(N.lib().pdmg_paradiag_rank_phase(self._h, k, C.byref(rep) if rep else None, sums))
            if k < 4:
                dist.barrier()
        t = torch.tensor([sums[0], sums[1]], dtype=torch.float64)
        if dist.get_backend() == "nccl":
            t = t.cuda()
        dist.all_reduce(t)
        rr, ff = float(t[0]), float(t[1])
        relres = (rr ** 0.5) / (ff ** 0.5) if ff > 0 else rr ** 0.5
        iters = it[self.t0:self.t0 + self.ntl].tolist() if want_iterations else None
        del H
        return iters, relres

    def close(self):
        if getattr(self, "_h", None):
            dist.barrier()  # peers close their mappings of our buffers before we free them
            self.N.lib().pdmg_paradiag_destroy(self._h)
            self._h = None
