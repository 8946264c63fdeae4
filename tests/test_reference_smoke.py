"""Drop-in proof with UNCHANGED reference callers (VERDICT r1 "next" 3).

The reference's own pytest (proj/python/tests/test_smoke.py, staged
byte-for-byte into oracle/_ref/tests/ by oracle/Makefile -- it is not in git)
runs against two `_paes` modules:
  * compat   -- paper_1403_7295_b200/compat/_paes.py, the engine's Python face;
  * patched  -- the reference's own pybind module (python/paes_module.cpp) and
                core sources, built by oracle/Makefile with
                oracle/patches/exec_gpu_chunk.patch applied, so its
                encrypt_chunk_into / decrypt_chunk_into (exec.cpp:111-127)
                call libpaes_cuda.so;
  * linked   -- the same unmodified module and core sources EXCEPT aes.cpp,
                compiled straight from the reference tree with NO patch and
                linked against lib/libpaes_aes_b200.so, which exports
                aes.hpp's symbols (encrypt_ecb, RoundKeySchedule, ...) over
                the engine: a link-level drop-in.
On a B200 all 7 non-CLI tests must pass (2 need the reference CLI and skip,
as they do in the reference's own run without PAES_CLI).  Without a GPU only
the host-only tests are run.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SMOKE = os.path.join(ROOT, "oracle", "_ref", "tests", "test_smoke.py")
MODULES = {
    "compat": os.path.join(ROOT, "paper_1403_7295_b200", "compat"),
    "patched": os.path.join(ROOT, "oracle", "_ref", "patched"),
    "linked": os.path.join(ROOT, "oracle", "_ref", "linked"),
}
HOST_ONLY = "test_key_schedule_shape or test_plan_chunks or test_reject_outliers"
# the library the reference modules link (their rpath), whatever PAES_CUDA_LIB
# points this process at (e.g. the coverage variant)
LINKED_LIB = os.path.join(ROOT, "paper_1403_7295_b200", "lib", "libpaes_cuda.so")


def _staged():
    if not os.path.exists(SMOKE):
        pytest.fail("oracle/_ref/tests/test_smoke.py is not staged: run `make -C oracle` where /root/reference exists")
    for which in ("patched", "linked"):
        if not os.path.isdir(MODULES[which]) or not any(f.startswith("_paes") for f in os.listdir(MODULES[which])):
            pytest.fail(f"oracle/_ref/{which}/_paes*.so is not built: run `make -C oracle`")


def _run_smoke(tmp_path, which: str, select: str | None = None):
    d = tmp_path / "smoke"
    d.mkdir()
    shutil.copy(SMOKE, d / "test_smoke.py")
    env = dict(os.environ, PYTHONPATH=MODULES[which])
    env.pop("PAES_CLI", None)
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "--rootdir", str(d), str(d / "test_smoke.py")]
    if select:
        cmd += ["-k", select]
    r = subprocess.run(cmd, cwd=str(d), env=env, capture_output=True, text=True, timeout=600)
    return r.returncode, r.stdout + r.stderr


@pytest.mark.parametrize("which", ["compat", "patched", "linked"])
def test_reference_smoke_host_only_tests(tmp_path, which):
    _staged()
    rc, out = _run_smoke(tmp_path, which, HOST_ONLY)
    assert rc == 0 and "3 passed" in out, out


@pytest.mark.gpu
@pytest.mark.parametrize("which", ["compat", "patched", "linked"])
def test_reference_smoke_unchanged_on_b200(tmp_path, which, gpu):
    _staged()
    rc, out = _run_smoke(tmp_path, which)
    assert rc == 0 and "7 passed, 2 skipped" in out, out


@pytest.mark.gpu
@pytest.mark.parametrize("which", ["patched", "linked"])
def test_reference_module_runs_the_gpu_engine(tmp_path, gpu, orc, which):
    """The reference module's encrypt_bytes / decrypt_bytes (paes_module.cpp:84-93
    -> encrypt_chunk -> encrypt_chunk_into -> [patched: paes_cuda_chunk |
    linked: aes::encrypt_ecb from libpaes_aes_b200.so]) launch libpaes_cuda.so
    kernels and match the reference's CPU bytes; a wrong key is the module's
    PaddingError."""
    snippet = r"""
import ctypes, json, os, sys
import _paes
key = bytes(range(16))
data = os.urandom((3 << 20) + 5)
lib = ctypes.CDLL(sys.argv[1])
lib.paes_cuda_launch_count.restype = ctypes.c_uint64
before = lib.paes_cuda_launch_count()
ct = _paes.encrypt_bytes(data, key)
assert _paes.decrypt_bytes(ct, key) == data
try:
    _paes.decrypt_bytes(ct, bytes(16))
    bad = "no error"
except ValueError as e:
    bad = type(e).__name__
maps = open("/proc/self/maps").read()
print(json.dumps({"launches": lib.paes_cuda_launch_count() - before, "bad": bad, "len": len(ct),
                  "loaded": "libpaes_cuda.so" in maps, "module": _paes.__file__}))
open(sys.argv[2], "wb").write(data + ct)
"""
    _staged()
    blob = tmp_path / "blob.bin"
    env = dict(os.environ, PYTHONPATH=MODULES[which])
    r = subprocess.run([sys.executable, "-c", snippet, os.path.realpath(LINKED_LIB), str(blob)], env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    import json

    info = json.loads(r.stdout.strip().splitlines()[-1])
    assert info["module"].startswith(MODULES[which]), info
    assert info["loaded"] and info["launches"] >= 3, info
    assert info["bad"] == "PaddingError", info
    raw = blob.read_bytes()
    n = (3 << 20) + 5
    assert raw[n:] == orc.encrypt_chunk(raw[:n], True, bytes(range(16)))


@pytest.mark.gpu
@pytest.mark.parametrize("strategy,workers", [("sequential", 1), ("threads", 4), ("threads", 16), ("processes", 3)])
def test_linked_reference_run_job_on_b200(tmp_path, gpu, orc, strategy, workers):
    """The reference's own run_job (exec.cpp:143-338, reached through its
    unmodified encrypt_file / decrypt_file, paes_module.cpp:121-149), compiled
    from its sources without aes.cpp: every chunk's aes::encrypt_ecb /
    decrypt_ecb is the engine's.  Outputs equal the oracle's, the round trip
    restores the input, kernels launched in-process (sequential / threads) or
    in the GPU worker (processes: worker_exe = lib/paes_gpu_worker, which the
    reference's process strategy spawns per chunk)."""
    snippet = r"""
import ctypes, json, sys
import _paes
lib = ctypes.CDLL(sys.argv[1])
lib.paes_cuda_launch_count.restype = ctypes.c_uint64
src, enc, dec, strategy, workers, exe = sys.argv[2:8]
key = bytes(range(16))
before = lib.paes_cuda_launch_count()
a = _paes.encrypt_file(src, enc, key, int(workers), strategy, exe)
b = _paes.decrypt_file(enc, dec, key, int(workers), strategy, exe)
try:
    _paes.decrypt_file(enc, dec + ".bad", bytes(16), int(workers), strategy, exe)
    bad = "no error"
except (ValueError, RuntimeError) as e:  # PaddingError / WorkerError
    bad = type(e).__name__
print(json.dumps({"launches": lib.paes_cuda_launch_count() - before, "enc": a, "dec": b, "bad": bad}))
"""
    _staged()
    n = (5 << 20) + 7
    data = os.urandom(n)
    src, enc, dec = tmp_path / "in.bin", tmp_path / "in.enc", tmp_path / "in.dec"
    src.write_bytes(data)
    exe = os.path.join(ROOT, "paper_1403_7295_b200", "lib", "paes_gpu_worker") if strategy == "processes" else ""
    env = dict(os.environ, PYTHONPATH=MODULES["linked"])
    r = subprocess.run([sys.executable, "-c", snippet, os.path.realpath(LINKED_LIB), str(src), str(enc),
                        str(dec), strategy, str(workers), exe], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    import json

    info = json.loads(r.stdout.strip().splitlines()[-1])
    assert enc.read_bytes() == orc.encrypt_chunk(data, True, bytes(range(16)))
    assert dec.read_bytes() == data
    assert not (tmp_path / "in.dec.bad").exists()
    # sequential: PaddingError (a ValueError); parallel strategies: WorkerError (a RuntimeError)
    assert info["bad"] == ("PaddingError" if strategy == "sequential" else "WorkerError"), info
    if strategy != "processes":
        assert info["launches"] >= 2, info
