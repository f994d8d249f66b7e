"""The C++ facade (include/pdmg_b200.hpp) compiles against the C ABI and behaves like the reference API."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "test_facade")


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
