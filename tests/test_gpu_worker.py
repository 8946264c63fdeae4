"""The GPU worker speaks the reference's hidden worker protocol, so the
reference's own, unmodified process strategy (run_process_isolated,
exec.cpp:272-338) runs on the B200 when worker_exe points at it."""
import os
import random
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def worker_path():
    from paper_1403_7295_b200 import build

    return build.WORKER


def test_worker_rejects_bad_arguments(lib):
    exe = worker_path()
    assert os.path.exists(exe)
    assert subprocess.run([exe], capture_output=True).returncode == 2
    r = subprocess.run([exe, "__worker", "--in", "x", "--out", "y", "--final", "1", "--dir", "sideways",
                        "--keyfd", "0"], capture_output=True, text=True)
    assert r.returncode == 2 and "bad --dir" in r.stderr


@pytest.mark.gpu
def test_reference_process_strategy_drives_gpu_workers(paes, gpu, ref, orc, tmp_path):
    rnd = random.Random(29)  # deterministic: the wrong-key check must not flake on a valid random trailer
    key = rnd.randbytes(16)
    data = rnd.randbytes(300_007)
    src = tmp_path / "p.bin"
    src.write_bytes(data)
    exe = worker_path()
    # reference run_job(ProcessIsolated, 3 workers) with the GPU worker binary
    rc, bi, bo, _ = ref.run_job(str(src), str(tmp_path / "c.bin"), key, 3, 2, 0, exe)
    assert rc == 0 and bi == len(data) and bo == (len(data) // 16 + 1) * 16
    assert (tmp_path / "c.bin").read_bytes() == orc.encrypt_chunk(data, True, key)
    rc, _, bo, _ = ref.run_job(str(tmp_path / "c.bin"), str(tmp_path / "d.bin"), key, 4, 2, 1, exe)
    assert rc == 0 and bo == len(data) and (tmp_path / "d.bin").read_bytes() == data
    # wrong key: the final worker fails, the reference aggregates a WorkerError, no output
    bad = bytes([key[0] ^ 1]) + key[1:]
    rc, _, _, _ = ref.run_job(str(tmp_path / "c.bin"), str(tmp_path / "bad.bin"), bad, 4, 2, 1, exe)
    assert rc == -1001
    assert not (tmp_path / "bad.bin").exists()
