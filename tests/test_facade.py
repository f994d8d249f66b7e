"""The C++ facade (include/pdmg_b200.hpp) compiles against the C ABI and behaves like the reference API."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "test_facade")
MULTI = os.path.join(ROOT, "tests", "cpp", "test_multi")


@pytest.fixture(scope="module")
def facade_bin():
    subprocess.run(["g++", "-std=c++17", "-O2", f"-I{ROOT}/include", f"{ROOT}/tests/cpp/test_facade.cpp",
                    f"-L{ROOT}/paper_2203_11154_b200", "-lpdmg_b200",
                    f"-Wl,-rpath,{ROOT}/paper_2203_11154_b200", "-o", BIN], check=True)
    return BIN


def test_facade_host_checks(facade_bin):
    out = subprocess.run([facade_bin], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    assert "host checks) ok" in out.stdout


@pytest.mark.gpu
def test_facade_gpu(facade_bin):
    out = subprocess.run([facade_bin, "--gpu"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "facade ok: C1 11 cycles, W(1,0) 14 cycles" in out.stdout


@pytest.fixture(scope="module")
def multi_bin():
    subprocess.run(["g++", "-std=c++17", "-O2", "-pthread", f"-I{ROOT}/include", f"{ROOT}/tests/cpp/test_multi.cpp",
                    f"-L{ROOT}/paper_2203_11154_b200", "-lpdmg_b200",
                    f"-Wl,-rpath,{ROOT}/paper_2203_11154_b200", "-o", MULTI], check=True)
    return MULTI


def test_multi_builds(multi_bin):
    assert os.path.exists(multi_bin)


@pytest.mark.gpu
def test_multi_context_and_device_list(multi_bin):
    """Two contexts from two host threads, and one context sharded over the device list {0, 0}: bitwise equal to
    one single-device context (proj/src/paradiag.cpp:207-236 chunking, test_paradiag.cpp:250-259 threads-bitwise)."""
    out = subprocess.run([multi_bin], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "multi ok" in out.stdout
