"""Build tests/cpp/test_shim.cpp against include/paes_gpu.hpp + libpaes_cuda.so
and run it: host mode here, gpu mode on a B200."""
from __future__ import annotations

import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def shim_exe(lib, tmp_path_factory):
    from paper_1403_7295_b200 import _native

    libdir = os.path.dirname(_native.lib_path())
    exe = str(tmp_path_factory.mktemp("shim") / "test_shim")
    cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
    cmd = [cxx, "-std=c++20", "-O1", "-Wall", "-Wextra", f"-I{ROOT}/include",
           os.path.join(ROOT, "tests", "cpp", "test_shim.cpp"), "-o", exe, f"-L{libdir}", "-lpaes_cuda",
           f"-Wl,-rpath,{libdir}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_cpp_shim_host(shim_exe):
    r = subprocess.run([shim_exe, "host"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_shim_gpu(shim_exe, gpu):
    r = subprocess.run([shim_exe, "gpu"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
