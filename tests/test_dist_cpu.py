"""Multi-rank path on CPU (gloo, world_size 2): shift sharding + max/sum reductions reproduce the single-
process batch exactly (paradiag.cpp:217-236 semantics: results independent of the worker count)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2203_11154_b200.sharding import reduce_scalar, shard

N, S = 32, 7


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys

    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from oracle_lib import Cfg, Oracle

    o = Oracle()
    lams = o.circulant_shifts(0.01, 32, 1 / 32, 0, S)
    b = o.random_complex(1, S * (N - 1) ** 2).reshape(S, N - 1, N - 1)
    b0, b1 = shard(S, rank, world)
    r = o.solve_batch(N, lams[b0:b1], Cfg(), b[b0:b1], threads=1)
    np.save(os.path.join(outdir, f"u{rank}.npy"), r["u"])
    np.save(os.path.join(outdir, f"it{rank}.npy"), r["iterations"])
    tmax = reduce_scalar(float(rank + 1), "max")
    tsum = reduce_scalar(float(b1 - b0), "sum")
    np.save(os.path.join(outdir, f"red{rank}.npy"), np.array([tmax, tsum]))
    dist.destroy_process_group()


def test_shard_covers_and_is_contiguous():
    for Sx in (1, 7, 256, 1024):
        for P in (1, 2, 3, 4, 8):
            parts = [shard(Sx, r, P) for r in range(P)]
            assert parts[0][0] == 0 and parts[-1][1] == Sx
            for (a0, a1), (c0, c1) in zip(parts, parts[1:]):
                assert a1 == c0
    assert shard(256, 3, 8) == (96, 128)
    with pytest.raises(ValueError):
        shard(8, 2, 2)


def test_two_rank_gloo_matches_single_process(tmp_path, oracle):
    from oracle_lib import Cfg

    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    u = np.concatenate([np.load(tmp_path / "u0.npy"), np.load(tmp_path / "u1.npy")])
    it = np.concatenate([np.load(tmp_path / "it0.npy"), np.load(tmp_path / "it1.npy")])
    lams = oracle.circulant_shifts(0.01, 32, 1 / 32, 0, S)
    b = oracle.random_complex(1, S * (N - 1) ** 2).reshape(S, N - 1, N - 1)
    ref = oracle.solve_batch(N, lams, Cfg(), b, threads=1)
    assert np.array_equal(u, ref["u"]) and np.array_equal(it, ref["iterations"])
    for r in range(2):
        tmax, tsum = np.load(tmp_path / f"red{r}.npy")
        assert tmax == 2.0 and tsum == S
