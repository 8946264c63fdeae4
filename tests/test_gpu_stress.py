"""tests/cpp/stress_threads.cpp against the product library: 8 threads x 40
mixed operations (pageable / pinned / zero-copy / device-pointer transforms,
host batches, file jobs, state transforms, runtime reconfiguration) under
concurrency, every result checked by round trip.  The same driver runs under
ThreadSanitizer via scripts/sanitizer_stress.sh (profiles/r01_tsan_stress.log)."""
from __future__ import annotations

import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_threaded_stress(lib, gpu, tmp_path):
    from paper_1403_7295_b200 import _native

    libdir = os.path.dirname(_native.lib_path())
    exe = str(tmp_path / "stress_threads")
    cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
    cmd = [cxx, "-std=c++17", "-O2", f"-I{ROOT}/include", "-I/usr/local/cuda/include",
           os.path.join(ROOT, "tests", "cpp", "stress_threads.cpp"), "-o", exe, f"-L{libdir}", "-lpaes_cuda",
           "-L/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{libdir}", "-Wl,-rpath,/usr/local/cuda/lib64"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([exe, "8", "40"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr[-4000:]
    assert "0 failures" in r.stdout
