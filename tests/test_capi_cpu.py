"""CPU tests of the C ABI boundary (no GPU): the library loads, exports every entry point the header
declares, validates configurations with the reference's error taxonomy and messages BEFORE touching
CUDA, and its host helpers reproduce the reference input generators."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2203_11154_b200 as P
from paper_2203_11154_b200 import _native as N


def header_functions():
    src = open(N.HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pdmg_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = N.lib()
    names = header_functions()
    assert len(names) >= 25
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert lib.pdmg_abi_version() == 2


def test_library_is_sm100a_fatbin():
    """The shipped .so carries sm_100a SASS (built with -gencode arch=compute_100a,code=sm_100a)."""
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", N.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_default_config_matches_reference():
    c = N.MgConfig()
    N.lib().pdmg_mg_config_default(C.byref(c))
    # multigrid.hpp:14-23, smoother.hpp:32-36
    assert (c.cycle, c.nu1, c.nu2, c.coarsest_n, c.tol, c.max_iter, c.smoother) == (1, 1, 0, 8, 1e-8, 200, 0)
    assert c.omega == 24.0 / 25.0
    d = P.MultigridConfig()
    assert (int(d.cycle), d.nu1, d.nu2, d.coarsest_n, d.tol, d.max_iter) == (1, 1, 0, 8, 1e-8, 200)


def test_random_rhs_matches_oracle(oracle):
    assert np.array_equal(P.random_rhs(64, 0).ravel(), oracle.random_complex(0, 63 * 63))
    many = P.random_rhs(16, 1, count=3)
    assert np.array_equal(many.ravel(), oracle.random_complex(1, 3 * 225))


def test_circulant_shifts_match_oracle(oracle):
    for a, nt, dt in ((0.01, 32, 1 / 32), (1e-3, 256, 1 / 256), (0.01, 1024, 2.0 ** -20)):
        np.testing.assert_allclose(P.circulant_shifts(a, nt, dt), oracle.circulant_shifts(a, nt, dt),
                                   rtol=1e-14, atol=1e-12)


@pytest.mark.parametrize("kw,msg", [
    (dict(nu1=-1), "negative smoothing counts"),
    (dict(nu1=0, nu2=0), "nu1 \\+ nu2 must be positive"),
    (dict(coarsest_n=1), "coarsest_n must be >= 2"),
    (dict(tol=0.0), "tol must be positive"),
    (dict(max_iter=0), "max_iter must be >= 1"),
    (dict(coarsest_n=5), "coarsening from n = 64 reaches n = 4, not coarsest_n = 5"),
    (dict(coarsest_n=128), "fine grid n = 64 is finer than coarsest_n = 128 allows"),
])
def test_config_errors_without_gpu(kw, msg):
    """multigrid.hpp:25-31 and multigrid.cpp:27-44 messages, raised as ConfigError before any CUDA call."""
    with pytest.raises(P.ConfigError, match=msg):
        P.BatchedMultigridHierarchy(P.Grid2D(64), [0.0], P.MultigridConfig(**kw))


def test_grid_errors():
    with pytest.raises(P.ConfigError, match="at least 2 subdivisions"):
        P.Grid2D(1)
    with pytest.raises(P.ConfigError, match="cannot be coarsened"):
        P.BatchedMultigridHierarchy(P.Grid2D(12), [0.0], P.MultigridConfig(coarsest_n=2))
    with pytest.raises(P.ConfigError, match="dense assembly refused for n = 130"):
        P.BatchedMultigridHierarchy(P.Grid2D(260), [0.0], P.MultigridConfig(coarsest_n=130))


def test_singular_smoother_at_construction():
    """multigrid.cpp:47-58: a singular Vanka patch fails at construction naming the level."""
    with pytest.raises(P.SingularOperatorError, match=r"level 1 \(n = 32\): vanka_coeffs: patch eigenvalue 2\+eta"):
        P.BatchedMultigridHierarchy(P.Grid2D(64), [-2 * 32 * 32], P.MultigridConfig(P.CycleKind.V, 1, 1, 4))
    with pytest.raises(P.SingularOperatorError, match="jacobi_weight: 4\\+eta"):
        P.BatchedMultigridHierarchy(P.Grid2D(64), [-4 * 64 * 64],
                                    P.MultigridConfig(smoother=P.SmootherConfig.jacobi()))


def test_no_gpu_is_a_loud_runtime_error():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(P.DeviceError):
        P.BatchedMultigridHierarchy(P.Grid2D(16), [0.0], P.MultigridConfig())


def test_shape_mismatch_is_config_error():
    """residual: grid mismatch (grid.cpp:93) -> ConfigError, checked on the host side of the boundary."""
    with pytest.raises(P.ConfigError, match="grid mismatch"):
        P.multigrid._as_batch(np.zeros((4, 4)), 1, 7, "MultigridHierarchy::solve")
