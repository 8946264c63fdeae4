"""Build tests/c/test_abi.c with gcc -std=c99 against include/paes_cuda.h
and libpaes_cuda.so: the boundary is usable from plain C."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def c_exe(lib, tmp_path_factory):
    from paper_1403_7295_b200 import _native

    libdir = os.path.dirname(_native.lib_path())
    exe = str(tmp_path_factory.mktemp("cabi") / "test_abi")
    cc = "/usr/bin/gcc" if os.path.exists("/usr/bin/gcc") else "gcc"
    r = subprocess.run([cc, "-std=c99", "-O1", "-Wall", "-Wextra", "-pedantic", f"-I{ROOT}/include",
                        os.path.join(ROOT, "tests", "c", "test_abi.c"), "-o", exe, f"-L{libdir}", "-lpaes_cuda",
                        f"-Wl,-rpath,{libdir}"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert "warning" not in r.stderr, r.stderr
    return exe


def test_c_abi_host(c_exe):
    r = subprocess.run([c_exe, "host"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_c_abi_gpu(c_exe, gpu):
    r = subprocess.run([c_exe, "gpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
