"""The C++ drop-in (include/pbh_gpu.hpp) compiles like reference test code and
its reference-restated assertions pass on the B200 (tests/cpp/test_shim.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def build(out):
    lib = os.path.join(ROOT, "paper_1908_09378_b200")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_shim.cpp"), "-L" + lib, "-lpbh_gpu",
                    "-Wl,-rpath," + lib, "-o", out], check=True)


def test_shim_compiles(tmp_path):
    build(str(tmp_path / "test_shim"))


@pytest.mark.gpu
def test_shim_runs_on_device(tmp_path):
    exe = str(tmp_path / "test_shim")
    build(exe)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.startswith("ok ")
