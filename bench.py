#!/usr/bin/env python3
"""Benchmark: batched complex-shifted-Laplacian multigrid solves on B200 (BASELINE.json metric).

A "step" is one full batched solve (every shift to relative residual 1e-10) of the workload's shifts.
Default workload = BASELINE config 3: h=1/512 (511x511 interior), n=256 shifts
lambda_j = (1 - alpha^(1/n) e^(2 pi i j/n))/dt with alpha=1e-3, dt=1/256, RHS uniform[-1,1]^2 from
std::mt19937(2) drawn shift-major, V(2,2) Vanka cycles (omega = 24/25), coarsest 3x3, complex128.
N>1 (torchrun): by default (`--scaling strong`) the config's batch is sharded contiguously over the ranks
(paradiag.cpp:217-236 chunking), as BASELINE config 3 words it; `--scaling weak` instead has every rank solve
its own full batch of the config's shifts (rank r's RHS from mt19937(seed + 100 r)).  Either way there is no
data-path collective, so `value` = all ranks' updates / max-over-ranks time.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl b200|reference]

Prints ONE JSON line (rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

CONFIGS = {
    # name: (n, n_shifts, alpha, n_t, dt, seed, nu1, nu2, description)
    "c1": (64, 1, 0.01, 32, 1 / 32, 0, 1, 1, "C1: n=64 (63x63), 1 shift (j=3 of n_t=32, alpha=0.01, dt=1/32), V(1,1), seed 0"),
    "c2": (128, 32, 0.01, 32, 1 / 32, 1, 1, 1, "C2: n=128 (127x127), 32 shifts (alpha=0.01, dt=1/32), V(1,1), seed 1"),
    "c3": (512, 256, 1e-3, 256, 1 / 256, 2, 2, 2,
           "C3: n=512 (511x511), 256 shifts (alpha=1e-3, dt=1/256), V(2,2), seed 2"),
    "c4a": (1024, 1024, 0.01, 1024, 1 / 1024, 3, 1, 1,
            "C4 set A: n=1024 (1023x1023), 1024 shifts (alpha=0.01, dt=1/1024), V(1,1), seed 3"),
    "c4b": (1024, 1024, 0.01, 1024, 2.0 ** -20, 3, 1, 1,
            "C4 set B: n=1024 (1023x1023), 1024 shifts (alpha=0.01, dt=h^2), V(1,1), seed 3"),
    "c5": (256, 256, 0.01, 256, 1 / 256, 4, 1, 1,
           "C5: ParaDIAG backward-Euler heat step, n=256 (255x255), nt=256 (T=1), alpha=0.01, V(1,1), "
           "IC sin(pi x)sin(pi y)+U[-0.1,0.1] seed 4; time DFT + 256 shifted solves + inverse DFT + residual"),
}
METRIC = "complex grid-point smoother updates/sec"
UNIT = "updates/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--c5-transport", default="ipc", choices=["ipc", "nccl"],
                    help="C5 on N>1 ranks: fused peer-memory transforms over CUDA IPC (default) or NCCL all-to-all")
    ap.add_argument("--shifts", type=int, default=0, help="override the number of shifts (0 = config's)")
    ap.add_argument("--nu", default="", help="override the cycle's nu1,nu2 (experiments; not a BASELINE config)")
    ap.add_argument("--precision", default="c128", choices=["c128", "c64"],
                    help="c64: fp32 storage / fp64 arithmetic, tol 1e-5 (BASELINE config 4)")
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"],
                    help="N>1: weak = every rank solves its own full batch of the config (rank r's RHS from "
                         "mt19937(seed + 100 r)); strong = the config's batch is split over the ranks")
    return ap.parse_args()


def dist_backend(local: int):
    """NCCL over NVLink; gloo for the one-GPU script-path tests (NCCL refuses two ranks on one device)."""
    import torch

    if os.environ.get("PDMG_BENCH_ONE_DEVICE"):
        return {"backend": "gloo"}
    return {"backend": "nccl", "device_id": torch.device("cuda", local)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("PDMG_BENCH_ONE_DEVICE"):  # script-path tests on a one-GPU box (never a reported number)
        local = 0
    return rank, world, local


def updates_per_cycle(n: int, nu1: int, nu2: int, coarsest: int = 4) -> float:
    tot, g = 0.0, n
    while g > coarsest:
        tot += (nu1 + nu2) * (g - 1) ** 2
        g //= 2
    return tot


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region (B200_PROFILING.md clocks line), in-process
    through NVML (the library nvidia-smi reads; spawning nvidia-smi every 50 ms contends for driver locks with the
    solve's per-cycle host synchronisation).  Falls back to nvidia-smi when NVML is unavailable."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40, "sw_power_cap": 0x4}

    def __init__(self, device: int, period_s: float = 0.02):
        self.device, self.period = device, period_s
        self.samples = []  # (sm_mhz, max_mhz, reasons_mask)
        self._stop = threading.Event()
        self.src = "nvml"

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def run():
                while not self._stop.is_set():
                    try:
                        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.samples.append((sm, mx, rs))
                    except Exception:
                        pass
                    self._stop.wait(self.period)

            self.thread = threading.Thread(target=run, daemon=True)
            self.thread.start()
        except Exception:
            self.thread = None
            self.src = "unavailable"
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self.thread:
            self.thread.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [f"clock sampling {self.src}"], "samples": 0}
        sm = [s[0] for s in self.samples]
        reasons = sorted({k for s in self.samples for k, bit in self.REASONS.items() if s[2] & bit})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(s[1] for s in self.samples), "reasons": reasons,
                "samples": len(self.samples), "source": self.src}


def roofline_of(stats: dict, config: str, upd_per_step: float, nu_sum: int) -> dict:
    """Roofline entry of the dominant kernel class (by CUDA-event time in the profiled pass).  `achieved` = SURVEY
    8(d) algorithmic bytes (48 B per c128 grid-point smoother update, 24 B c64, plus S/4 per point for a fused
    restriction / prolongation; a transform or residual pass: the bytes it must move) / the class's average launch
    time, against MEASURED_PEAKS.json hbm_gbs."""
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except Exception:
        pass
    peak = peaks.get("hbm_gbs")
    peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if peak else "fallback (B200_PROFILING.md 6650 GB/s)"
    peak = peak or 6650.0
    top_name, top = max(stats.items(), key=lambda kv: kv[1]["ms"])
    total_ms = sum(v["ms"] for v in stats.values())
    all_bytes = sum(v.get("unit_bytes", v["bytes"]) for v in stats.values())
    moved = None
    if top["bytes"] > 0:
        ub = top.get("unit_bytes") or top["bytes"]
        achieved = ub / (top["ms"] / 1e3) / 1e9
        mv = top["bytes"] / (top["ms"] / 1e3) / 1e9
        moved = {"moved_bytes_per_launch": top["bytes"] / top["launches"], "moved_GBps": round(mv, 1),
                 "moved_frac": round(mv / peak, 4), "updates_per_launch": top.get("updates", 0.0) / top["launches"]}
        bound = "hbm"
    else:
        # one-CTA-per-shift solve (small grids): its working set is L2/L1-resident, so report the
        # operator-level algorithmic bytes (96 B/update V(1,1), 72 B/update V(2,2), c128)
        bpu = {2: 96.0, 4: 72.0}.get(nu_sum, 96.0)
        achieved = upd_per_step * bpu / (top["ms"] / top["launches"] / 1e3) / 1e9
        bound = "latency (L2-resident working set; operator-level bytes)"
    roofline = {"bound": bound, "kernel": top_name, "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": None, "peak_source": peak_src,
                "kernel_share_of_step": round(top["ms"] / total_ms, 4),
                "timing": "per-kernel CUDA events on the library stream, profiled pass right after the timed region",
                "launch_avg_ms": round(top["ms"] / top["launches"], 4),
                "algo_bytes_per_launch": (top.get("unit_bytes") or top["bytes"]) / top["launches"],
                "algo_bytes_def": "SURVEY 8(d): 48 B (c128) / 24 B (c64) per grid-point smoother update, plus "
                                  "S/4 per point for a fused restriction or prolongation",
                "all_kernels_algorithmic_GBps": round(all_bytes / (total_ms / 1e3) / 1e9, 1),
                "frac_note": "a two-sweep pass performs two smoother updates per point while streaming the level "
                             "once (temporal blocking), so its SURVEY 8(d) algorithmic rate can exceed the HBM "
                             "peak; moved_GBps / moved_frac are the bytes the pass physically moves"}
    if moved:
        roofline.update(moved)
    roofline.update(traffic_for(config, top_name))
    return roofline


def kernels_summary(stats: dict, top: int = 12) -> dict:
    return {k: {"launches": v["launches"], "ms": round(v["ms"], 3),
                "GBps": round(v.get("unit_bytes", v["bytes"]) / v["ms"] / 1e6, 1) if v["ms"] > 0 else None,
                "moved_GBps": round(v["bytes"] / v["ms"] / 1e6, 1) if v["ms"] > 0 else None}
            for k, v in sorted(stats.items(), key=lambda kv: -kv[1]["ms"])[:top]}


def so_sha16() -> str:
    """Identity of the running build: the hash of the library's sources (a rebuilt .so is not byte-identical)."""
    from paper_2203_11154_b200 import _native as N

    return N.source_sha16()


def traffic_for(config: str, kernel: str) -> dict:
    """ncu DRAM traffic per launch of `kernel` (dram__bytes_read.sum + dram__bytes_write.sum, one `ncu --set full`
    capture, profiles/traffic.json).  Each capture is stamped with the sha256 of the library sources it was built from;
    a capture of another build is not reported as this build's traffic."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tj = json.load(f)
    except Exception:
        return {"traffic": None, "traffic_note": "no ncu capture in profiles/traffic.json"}
    ent = tj.get(config, {}).get(kernel)
    if not isinstance(ent, dict):
        return {"traffic": None, "traffic_note": f"no ncu capture of {kernel} for {config}"}
    cur = so_sha16()
    if ent.get("src_sha16", ent.get("so_sha16")) != cur:
        return {"traffic": None, "traffic_note": f"ncu capture is of build {ent.get('src_sha16', ent.get('so_sha16'))}, this build is {cur}",
                "traffic_stale": ent.get("bytes")}
    return {"traffic": ent["bytes"], "traffic_source": ent.get("source", "profiles/traffic.json"),
            "traffic_build": cur}


def cpu_reference_run(n, lams, nu1, nu2, b, threads, tol=1e-10):
    """Reference CPU path: the reference's own grid.cpp/smoother.cpp (oracle/_ref) when built, else the C port.
    Shifts split over `threads` std::threads in contiguous chunks (paradiag.cpp:217-236)."""
    from oracle_lib import Cfg, Oracle, RefLib

    cfg = Cfg(nu1=nu1, nu2=nu2, tol=tol)
    try:
        lib, kind = RefLib(), "reference"
    except (FileNotFoundError, OSError):
        lib, kind = Oracle(), "port"
    t = time.perf_counter()
    out = lib.solve_batch(n, lams, cfg, b, threads=threads)
    dt = time.perf_counter() - t
    return out, dt, kind


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_sample(n, lams_all, nu1, nu2, b_all, threads, budget_s, tol=1e-10):
    """Time a bounded, contiguous sample of the workload's shifts (the workload's own right-hand sides) on the
    host cores with `threads` std::threads, plus one shift on one core (T = nproc and T = 1).
    Returns the baseline record and the oracle's per-shift results for the parity check."""
    m = n - 1
    upc = updates_per_cycle(n, nu1, nu2)
    out1, t1, kind = cpu_reference_run(n, lams_all[:1], nu1, nu2, b_all[:1], 1, tol)  # one shift on one core
    count = int(max(threads, min(len(lams_all), threads * max(1, round(budget_s / max(t1, 1e-3))))))
    count = min(count, len(lams_all))
    out, dt, kind = cpu_reference_run(n, lams_all[:count], nu1, nu2, b_all[:count], threads, tol)
    upd = float(np.sum(out["iterations"])) * upc
    rec = dict(value=upd / dt, unit=UNIT, cores=threads, kind=kind, cpu_model=cpu_model(),
               sample=f"shifts 0..{count - 1} of the workload ({count} of {len(lams_all)}, the workload's own "
                      f"right-hand sides), {threads} std::threads, {dt:.2f} s wall",
               shifts_per_s=count / dt, seconds=dt,
               single_core={"value": float(out1["iterations"][0]) * upc / t1, "unit": UNIT, "cores": 1,
                            "sample": f"shift 0 on one core, {t1:.3f} s", "shifts_per_s": 1.0 / t1})
    return rec, out, count


def parity_block(reps, u_dev, cpu_out, count, tol):
    """GPU vs the CPU reference path on the same inputs (north_star: identical per-shift V-cycle counts, solution and
    residual history within 1e-10 relative): shifts 0..count-1 of the workload."""
    it_ref = np.asarray(cpu_out["iterations"][:count])
    it_gpu = np.array([r.iterations for r in reps[:count]])
    u_err = h_err = 0.0
    margin = np.inf
    for s in range(count):
        it = int(it_ref[s])
        h_ref = cpu_out["hist"][s, : it + 1]
        if h_ref[0] > 0:
            if it_gpu[s] == it:
                h_err = max(h_err, float(np.max(np.abs(reps[s].residual_history - h_ref)) / h_ref[0]))
            margin = min(margin, abs(h_ref[-1] / h_ref[0] - tol) / tol)
        ref_u = cpu_out["u"][s]
        u_err = max(u_err, float(np.linalg.norm((u_dev[s] - ref_u).ravel()) / max(np.linalg.norm(ref_u.ravel()), 1e-300)))
    return {"shifts_compared": int(count), "iters_equal": bool(np.array_equal(it_ref, it_gpu)),
            "iters_equal_count": int(np.sum(it_ref == it_gpu)), "max_rel_err_u": u_err,
            "max_rel_err_history": h_err, "min_stop_margin": float(margin),
            "reference": "oracle/_ref (the reference's own grid.cpp/smoother.cpp + restated driver) on the box's host"}


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return 0
    n, S, alpha, nt, dt, seed, nu1, nu2, desc = CONFIGS[args.config]
    from oracle_lib import Oracle

    o = Oracle()
    lams = o.circulant_shifts(alpha, nt, dt, 0, S)
    threads = os.cpu_count() or 1
    m = n - 1
    upc = updates_per_cycle(n, nu1, nu2)
    # per step: a bounded sample of `threads` shifts (one per core) of the workload itself -- its own shifts and
    # right-hand sides (the seed's shift-major stream) -- cycling through the shift list
    per = min(S, threads)
    if args.config == "c1":
        lams = o.circulant_shifts(alpha, nt, dt, 3, 1)
    b_all = o.random_complex(seed, S * m * m).reshape(S, m, m)
    vals, times, kind = [], [], "port"
    for step in range(args.warmup + args.steps):
        j0 = (step * per) % S
        idx = [(j0 + q) % S for q in range(per)]
        out, t, kind = cpu_reference_run(n, lams[idx], nu1, nu2, np.ascontiguousarray(b_all[idx]), threads)
        if step >= args.warmup:
            vals.append(float(np.sum(out["iterations"])) * upc / t)
            times.append(t)
    value = statistics.median(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(times),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": {"workload": desc, "sample_per_step": f"{per} shifts on {threads} host threads",
                   "same_inputs": "the workload's own shifts and seed-stream right-hand sides"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind, "cpu_model": cpu_model(),
                         "sample": f"{per} shifts per step (one per core) of {args.config}: the workload's own "
                                   "shifts and right-hand sides, cycling through the batch"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_paradiag(args):
    """C5: one full ParaDIAG step per bench step (alpha-scaled time DFT, the nt shifted multigrid solves,
    inverse DFT, all-at-once residual).  N>1 ranks shard time slices; NCCL all-to-all moves the data."""
    rank, world, local = dist_env()
    import torch

    import paper_2203_11154_b200 as P
    from paper_2203_11154_b200.paradiag import ParadiagCirculant, heat_initial_rhs

    torch.cuda.set_device(local)
    n, S, alpha, nt, dt, seed, nu1, nu2, desc = CONFIGS["c5"]
    cfg = P.MultigridConfig(P.CycleKind.V, nu1, nu2, 4, 1e-10, 200, P.SmootherConfig.vanka())
    m = n - 1
    f = heat_initial_rhs(n, nt, dt, seed)
    upc = updates_per_cycle(n, nu1, nu2)
    pdr = None
    if world > 1:
        import torch.distributed as dist

        from paper_2203_11154_b200.paradiag_dist import GpuOps, paradiag_step

        dist.init_process_group(**dist_backend(local))
        transport = args.c5_transport
        if transport == "ipc":
            # each rank owns its time slices in the library; peers' slice buffers are opened over CUDA IPC and the
            # time transforms gather / scatter across the ranks through NVLink peer memory inside the kernel
            try:
                from paper_2203_11154_b200.paradiag_dist import IpcParadiag

                pdr = IpcParadiag(n, nt, alpha, dt, cfg, local)
                ctype = {"shape": (pdr.ntl * m * m * 2,), "typestr": "<f8", "data": (pdr.f_ptr, False), "version": 3}
                fv = torch.as_tensor(type("DevView", (), {"__cuda_array_interface__": ctype})(), device=f"cuda:{local}")
                fv.copy_(torch.from_numpy(np.ascontiguousarray(f[pdr.t0:pdr.t0 + pdr.ntl]).view(np.float64).ravel()))
                torch.cuda.synchronize()
                def step():
                    it, rr = pdr.step()
                    return None, it, rr
            except Exception as e:  # fall back to the NCCL all-to-all driver
                print(f"bench: IPC transport unavailable ({e}); using NCCL all-to-all", file=sys.stderr)
                transport, pdr = "nccl", None
        if transport == "nccl":
            ntl = nt // world
            f_local = torch.from_numpy(f[rank * ntl:(rank + 1) * ntl].reshape(ntl, m * m).view(np.float64)
                                       .reshape(ntl, m * m, 2)).to(f"cuda:{local}")
            ops = GpuOps(n, nt, alpha, dt, cfg, local)
            step = lambda: paradiag_step(f_local, n, nt, alpha, dt, ops)  # noqa: E731
    else:
        pd = ParadiagCirculant(n, nt, alpha, dt, cfg, device=local)
        d_f = torch.from_numpy(f.view(np.float64)).to(f"cuda:{local}")
        d_u = torch.empty_like(d_f)
        step = lambda: (None, None, pd.run_device(d_f.data_ptr(), d_u.data_ptr()))  # noqa: E731
    for _ in range(args.warmup):
        out = step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    # events on the stream the library launches on (the solver's stream for one GPU, torch's for the
    # distributed driver whose kernels run on torch's current stream)
    from paper_2203_11154_b200 import _native as N

    sh = (N.lib().pdmg_stream(pd.solver_handle) if world == 1 else
          N.lib().pdmg_stream(pdr.solver_handle) if pdr is not None else None)
    stream = torch.cuda.ExternalStream(sh) if sh else torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world == 1:
        N.lib().pdmg_reset_stats(pd.solver_handle)
    t0 = time.perf_counter()
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            out = step()
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / args.steps
    wall_ms = (time.perf_counter() - t0) * 1e3 / args.steps
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=f"cuda:{local}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    relres = out[2]
    launches = int(N.lib().pdmg_launch_count(pd.solver_handle)) if world == 1 else None
    roofline, kern = None, None
    if world == 1:  # per-kernel CUDA events in a separate profiled pass (the timed region carries no events)
        from paper_2203_11154_b200.multigrid import kernel_stats

        hs = pd.solver_handle
        N.lib().pdmg_reset_stats(hs)
        N.lib().pdmg_set_profiling(hs, 1)
        for _ in range(max(1, min(args.steps, 3))):
            step()
        torch.cuda.synchronize()
        kst = kernel_stats(hs)
        N.lib().pdmg_set_profiling(hs, 0)
        roofline = roofline_of(kst, "c5", 0.0, nu1 + nu2)
        kern = kernels_summary(kst)
    # total V-cycles over all slots (for the updates count), from one reported run
    if world == 1:
        u, reps, rr = pd.run(f)
        iters_total = sum(r.iterations for r in reps)
    else:
        iters_total = float(sum(out[1]))
        t = torch.tensor([iters_total], dtype=torch.float64, device=f"cuda:{local}")
        torch.distributed.all_reduce(t)
        iters_total = float(t.item())
    value = iters_total * upc / (ms / 1e3)
    e2e = None
    if world == 1:
        # end to end through the host-buffer C ABI (pdmg_paradiag_run): pinned f in, pinned u out
        import ctypes

        nbytes = f.nbytes
        hf = N.lib().pdmg_host_alloc(nbytes)
        hu = N.lib().pdmg_host_alloc(nbytes)
        ctypes.memmove(hf, np.ascontiguousarray(f).ctypes.data, nbytes)
        rr = ctypes.c_double(0.0)
        st = N.lib().pdmg_paradiag_run(pd._h, hf, hu, None, ctypes.byref(rr))  # untimed first call
        assert st == 0, N.lib().pdmg_last_error()
        e_steps = max(1, min(args.steps, 3))
        t0 = time.perf_counter()
        for _ in range(e_steps):
            st = N.lib().pdmg_paradiag_run(pd._h, hf, hu, None, ctypes.byref(rr))
            assert st == 0, N.lib().pdmg_last_error()
        e_s = time.perf_counter() - t0
        N.lib().pdmg_host_free(hf)
        N.lib().pdmg_host_free(hu)
        e2e = {"value": e_steps * iters_total * upc / e_s, "unit": UNIT, "h2d_bytes_per_step": nbytes,
               "d2h_bytes_per_step": nbytes, "steps": e_steps, "ms_per_step": 1e3 * e_s / e_steps}
    cpu = parity = None
    if world == 1 and not args.no_cpu_baseline:
        try:  # the oracle's ParaDIAG (C restatement of paradiag.cpp:185-248 with the alpha-circulant transforms)
            from oracle_lib import Cfg, Oracle

            thr = os.cpu_count() or 1
            t_c = time.perf_counter()
            ref = Oracle().paradiag(n, nt, alpha, dt, Cfg(nu1=nu1, nu2=nu2), f, threads=thr)
            t_c = time.perf_counter() - t_c
            iters_ref = int(np.sum(ref["iterations"]))
            cpu = {"value": iters_ref * upc / t_c, "unit": UNIT, "cores": thr, "kind": "port", "cpu_model": cpu_model(),
                   "sample": f"the whole C5 step (time transforms + {nt} shifted solves + residual), {thr} threads, "
                             f"{t_c:.2f} s wall", "seconds": t_c}
            it_gpu = np.array([r.iterations for r in reps])
            parity = {"slots_compared": nt, "iters_equal": bool(np.array_equal(it_gpu, ref["iterations"])),
                      "max_rel_err_u": float(np.linalg.norm((u - ref["u"]).ravel()) / np.linalg.norm(ref["u"].ravel())),
                      "relres_gpu": relres, "relres_oracle": ref["relres"],
                      "reference": "oracle/liboracle.so (orc_paradiag_circulant) on the box's host"}
        except Exception as e:
            cpu = {"error": str(e)}
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "gpu_launches": launches, "cpu_baseline": cpu, "parity": parity,
            "vs_baseline": None, "dtype": "c128", "data": "synthetic",
            "config": {"workload": desc, "parallelism": f"time-sharded x{world}" + (
                "" if world == 1 else " + fused peer-memory (CUDA IPC) time transforms" if pdr is not None
                else " + NCCL all-to-all")},
            "paradiag_steps_per_s": 1e3 / ms, "relres": relres, "cycles_total": iters_total,
            "host_wall_ms_per_step": wall_ms, "e2e": e2e, "roofline": roofline, "kernels": kern,
            "clocks": clk.summary()}), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.config == "c5":
        return run_paradiag(args)
    rank, world, local = dist_env()
    import torch

    import paper_2203_11154_b200 as P
    from paper_2203_11154_b200.sharding import shard

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group(**dist_backend(local))
    n, S, alpha, nt, dt, seed, nu1, nu2, desc = CONFIGS[args.config]
    if args.shifts:
        S = args.shifts
    if args.nu:
        nu1, nu2 = (int(x) for x in args.nu.split(","))
        desc += f" [nu1,nu2 = {nu1},{nu2}]"
    m = n - 1
    weak = world > 1 and args.scaling == "weak"
    b0, b1 = (0, S) if weak else shard(S, rank, world)
    Sr = b1 - b0
    rhs_seed = seed + 100 * rank if weak else seed
    j0 = 3 if args.config == "c1" else 0  # BASELINE config 1 is slot j = 3 of the n_t = 32 family
    lams_all = P.circulant_shifts(alpha, nt, dt, j0, S)
    lams = lams_all[b0:b1]
    tol = 1e-5 if args.precision == "c64" else 1e-10
    cfg = P.MultigridConfig(P.CycleKind.V, nu1, nu2, 4, tol, 200, P.SmootherConfig.vanka())
    # inputs: one mt19937(seed) stream, shift-major; each rank keeps its shard
    b_all = P.random_rhs(n, rhs_seed, count=b1)
    b_host = np.ascontiguousarray(b_all.reshape(b1, m, m)[b0:b1])
    del b_all
    H = P.BatchedMultigridHierarchy(P.Grid2D(n), lams, cfg, device=local, precision=args.precision)
    stream = torch.cuda.ExternalStream(H.stream)
    d_b = torch.from_numpy(b_host.view(np.float64)).to(f"cuda:{local}")
    d_u = torch.empty_like(d_b)
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], device=f"cuda:{local}", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], device=f"cuda:{local}", dtype=torch.float64)
        torch.distributed.all_reduce(t)
        return float(t.item())

    # ---- warm-up ---------------------------------------------------------------------------
    reps = None
    for _ in range(args.warmup):
        reps = H.solve_device(d_b.data_ptr(), d_u.data_ptr())
    # ---- timed region: device-resident inputs, CUDA events on the library's stream ----------
    H.reset_stats()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        upd = 0.0
        for _ in range(args.steps):
            reps = H.solve_device(d_b.data_ptr(), d_u.data_ptr())
            upd += H.last_updates()
        ev1.record(stream)
        barrier()
    ms = ev0.elapsed_time(ev1)
    launches = H.launch_count()
    # ---- per-kernel CUDA-event timing (separate pass: per-launch events cost ~6% of a step) ----
    H.reset_stats()
    H.set_profiling(True)
    for _ in range(max(1, min(args.steps, 3))):
        H.solve_device(d_b.data_ptr(), d_u.data_ptr(), want_reports=False)
    torch.cuda.synchronize()
    stats = H.kernel_stats()
    H.set_profiling(False)
    ms_max = max_over_ranks(ms)
    upd_all = sum_over_ranks(upd)
    value = upd_all / (ms_max / 1e3)
    S_job = Sr * world if weak else S
    shifts_per_s = args.steps * S_job / (ms_max / 1e3)
    iters = [r.iterations for r in reps]
    conv = all(r.converged for r in reps)

    # ---- N > 1 strong scaling: also the weak-scaled companion (every rank solves its own full batch) ----------
    weak_extra = None
    if world > 1 and not weak:
        bw = P.random_rhs(n, seed + 100 * rank, count=S)
        Hw = P.BatchedMultigridHierarchy(P.Grid2D(n), lams_all, cfg, device=local, precision=args.precision)
        d_bw = torch.from_numpy(bw.reshape(S, m, m).view(np.float64)).to(f"cuda:{local}")
        d_uw = torch.empty_like(d_bw)
        del bw
        for _ in range(args.warmup):
            Hw.solve_device(d_bw.data_ptr(), d_uw.data_ptr(), want_reports=False)
        sw = torch.cuda.ExternalStream(Hw.stream)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(sw)
        upd_w = 0.0
        for _ in range(args.steps):
            Hw.solve_device(d_bw.data_ptr(), d_uw.data_ptr(), want_reports=False)
            upd_w += Hw.last_updates()
        e1.record(sw)
        barrier()
        ms_w = max_over_ranks(e0.elapsed_time(e1))
        weak_extra = {"value": sum_over_ranks(upd_w) / (ms_w / 1e3), "unit": UNIT, "ms_per_step": ms_w / args.steps,
                      "workload": f"every rank solves its own {S}-shift batch (rank r: RHS seed {seed} + 100 r)",
                      "scaling": "weak"}
        Hw.close()
        del d_bw, d_uw

    # ---- end to end through the host API: pinned host b -> device -> solve -> host u ----------
    import ctypes

    from paper_2203_11154_b200 import _native as N

    nbytes = b_host.nbytes
    hb = N.lib().pdmg_host_alloc(nbytes)
    hu = N.lib().pdmg_host_alloc(nbytes)
    ctypes.memmove(hb, b_host.ctypes.data, nbytes)
    e_steps = max(1, min(args.steps, 3))
    rep = N.SolveReport(0, 0, 0, 0, 0.0)
    # one untimed host-API call first: it creates the copy stream/events and touches the pinned pages
    st = N.lib().pdmg_solve(H._h, hb, hu, ctypes.byref(rep))
    assert st == 0, N.lib().pdmg_last_error()
    barrier()
    t0 = time.perf_counter()
    e_upd = 0.0
    for _ in range(e_steps):
        st = N.lib().pdmg_solve(H._h, hb, hu, ctypes.byref(rep))
        assert st == 0, N.lib().pdmg_last_error()
        e_upd += H.last_updates()
    barrier()
    e_s = time.perf_counter() - t0
    e_s_max = max_over_ranks(e_s)
    e_value = sum_over_ranks(e_upd) / e_s_max
    N.lib().pdmg_host_free(hb)
    N.lib().pdmg_host_free(hu)
    # the same through pageable host buffers (numpy arrays; what a std::vector through the C++ facade passes):
    # the library page-locks them for the call (cudaHostRegister) and runs the same chunked pipeline
    u_np = np.empty_like(b_host)
    st = N.lib().pdmg_solve(H._h, b_host.ctypes.data, u_np.ctypes.data, ctypes.byref(rep))
    assert st == 0, N.lib().pdmg_last_error()
    barrier()
    t0 = time.perf_counter()
    for _ in range(e_steps):
        st = N.lib().pdmg_solve(H._h, b_host.ctypes.data, u_np.ctypes.data, ctypes.byref(rep))
        assert st == 0, N.lib().pdmg_last_error()
    barrier()
    e_pg = max_over_ranks(time.perf_counter() - t0)
    e2e_pageable = {"value": sum_over_ranks(e_upd) / e_pg, "unit": UNIT, "ms_per_step": 1e3 * e_pg / e_steps,
                    "buffers": "pageable numpy arrays (through the library's pinned bounce buffers)"}
    del u_np

    roofline = roofline_of(stats, args.config, upd / args.steps, nu1 + nu2)
    cpu = parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            lam_np = np.asarray(lams_all, np.complex128)
            cpu, cpu_out, count = cpu_sample(n, lam_np, nu1, nu2, b_host, os.cpu_count() or 1, budget_s=10.0, tol=tol)
            u_s = d_u.view(S, m, m, 2)[:count].cpu().numpy()
            parity = parity_block(reps, u_s[..., 0] + 1j * u_s[..., 1], cpu_out, count, tol)
            if args.precision == "c64":
                parity["note"] = "complex64 (fp32 storage) vs the fp64 reference at the same tol: north_star bound 1e-4 on u"
        except Exception as e:  # the baseline is reported, never required for the GPU number
            cpu = {"error": str(e)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak" if weak else "strong", "vs_baseline": None, "dtype": args.precision,
            "data": "synthetic",
            "config": {"workload": desc + (f" [{S} shifts]" if args.shifts else "")
                       + (f" per rank (rank r: RHS seed {seed} + 100 r)" if weak else ""), "shifts": S_job,
                       "precision": args.precision + (" (fp32 storage, fp64 arithmetic), tol 1e-5"
                                                      if args.precision == "c64" else ", tol 1e-10"),
                       "shifts_per_rank": Sr, "parallelism": (f"independent {Sr}-shift batch per rank x{world}" if weak
                                       else f"shift-sharded x{world}"),
                       "l2": "inputs larger than L2 (each fine array %.2f GB)" % (S * (n + 1) * n * 16 / 1e9)
                       if S * (n + 1) * n * 16 > 126e6 else "working set fits in L2 (latency-bound config)"},
            "shifts_per_s": shifts_per_s, "cycles_per_shift": sorted(set(iters)), "all_converged": conv,
            "e2e": {"value": e_value, "unit": UNIT, "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
                    "steps": e_steps, "ms_per_step": 1e3 * e_s_max / e_steps,
                    "buffers": "pinned (pdmg_host_alloc)"},
            "e2e_pageable": e2e_pageable,
            "weak_scaling": weak_extra,
            "gpu_launches": int(launches),
            "roofline": roofline,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
            "parity": parity,
            "kernels": kernels_summary(stats),
        }
        print(json.dumps(line), flush=True)
    H.close()
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
