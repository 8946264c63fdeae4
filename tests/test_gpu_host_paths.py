"""The host-pointer paths of paes_cuda_chunk, each forced explicitly: the
zero-copy kernel on pinned buffers, the pinned direct ring (zero-copy off),
the double-buffered bounce path for pageable ranges up to 4 MiB and the staged ring for
pageable memory -- all bit-exact vs the oracle across piece boundaries, and
each rejecting a wrong key."""
import ctypes as C
import os
import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
MiB = 1 << 20


def _run(paes, direction, src_ptr, n, final, key, dst_ptr, expect_rc=0):
    from paper_1403_7295_b200 import _native as N

    olen = C.c_uint64()
    rc = N.load().paes_cuda_chunk(direction, src_ptr, n, int(final), paes.round_keys(key), dst_ptr, C.byref(olen), 1)
    assert rc == expect_rc, N.last_error()
    return olen.value


@pytest.mark.parametrize("mode", ["pinned_zero_copy", "pinned_ring", "pageable"])
def test_ring_paths_vs_oracle(paes, gpu, orc, mode):
    import torch

    pinned = mode != "pageable"
    paes.set_pipeline(64 * 1024, 3)  # tiny pieces: many slots in flight, small-path threshold 64 KiB
    paes.set_zero_copy_max(0 if mode == "pinned_ring" else paes.DEFAULT_ZERO_COPY_MAX)
    rnd = random.Random(hash(mode) & 0xFFFF)
    try:
        key = rnd.randbytes(16)
        bad = bytes([key[0] ^ 0x80]) + key[1:]
        for n in [100, 64 * 1024, 64 * 1024 + 1, 3 * 64 * 1024 + 7, 1_000_003]:
            data = rnd.randbytes(n)
            if pinned:
                src = torch.empty(n + 32, dtype=torch.uint8, pin_memory=True)
                dst = torch.empty(n + 32, dtype=torch.uint8, pin_memory=True)
                src[:n] = torch.frombuffer(bytearray(data), dtype=torch.uint8)
                sp, dp = src.data_ptr(), dst.data_ptr()
                read = lambda m: dst[:m].numpy().tobytes()  # noqa: E731
            else:
                src = np.frombuffer(bytearray(data) + bytearray(32), dtype=np.uint8)
                dst = np.zeros(n + 32, dtype=np.uint8)
                sp, dp = src.ctypes.data, dst.ctypes.data
                read = lambda m: dst[:m].tobytes()  # noqa: E731
            m = _run(paes, 0, sp, n, True, key, dp)
            want = orc.encrypt_chunk(data, True, key)
            assert m == len(want) and read(m) == want, (n, pinned)
            # decrypt back (in place in the output buffer)
            k = _run(paes, 1, dp, m, True, key, dp)
            assert k == n and read(n) == data, (n, pinned)
            # a wrong key fails the trailer check on this path too (EBADMSG)
            m = _run(paes, 0, sp, n, True, key, dp)
            try:
                expect = orc.decrypt_chunk(want, True, bad)
            except ValueError:
                expect = None
            if expect is None:
                _run(paes, 1, dp, m, True, bad, dp, expect_rc=-74)
            else:  # the wrong key happened to leave a valid trailer: same bytes as the oracle
                k = _run(paes, 1, dp, m, True, bad, dp)
                assert read(k) == expect
    finally:
        paes.set_pipeline(256 * MiB, 3)
        paes.set_zero_copy_max(paes.DEFAULT_ZERO_COPY_MAX)


def test_oversized_pipeline_fails_cleanly_and_recovers(paes, gpu, orc):
    """A staging ring too large for the device raises GpuError, leaves no
    half-built ring behind, and the next call with a sane pipeline works."""
    rnd = random.Random(77)
    key = rnd.randbytes(16)
    data = rnd.randbytes(5 * MiB + 5)  # pageable, > the 4 MiB bounce path: the staged ring
    try:
        paes.set_pipeline(16 << 30, 32)  # 32 x 16 GiB of device slots: cannot fit
        with pytest.raises(paes.GpuError):
            paes.encrypt_bytes(data, key)
        with pytest.raises(paes.GpuError):  # same config again: still a clean failure, no stale ring
            paes.encrypt_bytes(data, key)
    finally:
        paes.set_pipeline(256 * MiB, 3)
    assert paes.encrypt_bytes(data, key) == orc.encrypt_chunk(data, True, key)
    n = 2 * MiB
    hin = np.frombuffer(rnd.randbytes(n), dtype=np.uint8).copy()
    hout = np.zeros(n + 16, dtype=np.uint8)
    ol = paes.ecb_batch_host(0, hin.ctypes.data, hout.ctypes.data, [0], [0], [n], paes.round_keys(key), True)
    assert hout[: ol[0]].tobytes() == orc.encrypt_chunk(hin.tobytes(), True, key)


def test_batch_host_messages_larger_than_the_staging_chunk(paes, gpu, orc):
    """A message longer than the pipeline chunk gets its own stream-ordered
    device spans (batch_host's `fits == false` branch); neighbours stay in
    normal groups."""
    rnd = random.Random(5151)
    paes.set_pipeline(1 * MiB, 3)
    try:
        lens = [100, 3 * MiB + 5, 7, 2 * MiB, 4096]
        keys = [rnd.randbytes(16) for _ in lens]
        msgs = [rnd.randbytes(L) for L in lens]
        in_off, out_off, oi, oo = [], [], 0, 0
        for L in lens:
            in_off.append(oi)
            out_off.append(oo)
            oi += L + 3
            oo += (L // 16 + 1) * 16 + 5
        hin = np.zeros(oi, dtype=np.uint8)
        for o, m in zip(in_off, msgs):
            hin[o:o + len(m)] = np.frombuffer(m, dtype=np.uint8)
        hout = np.full(oo, 0x77, dtype=np.uint8)
        rks = b"".join(paes.round_keys(k) for k in keys)
        ol = paes.ecb_batch_host(0, hin.ctypes.data, hout.ctypes.data, in_off, out_off, lens, rks, True)
        for o, n, m, k in zip(out_off, ol, msgs, keys):
            assert hout[o:o + n].tobytes() == orc.encrypt_chunk(m, True, k)
        back = np.zeros(oo, dtype=np.uint8)
        dl = paes.ecb_batch_host(1, hout.ctypes.data, back.ctypes.data, out_off, out_off, ol, rks, True)
        assert [back[o:o + n].tobytes() for o, n in zip(out_off, dl)] == msgs
    finally:
        paes.set_pipeline(256 * MiB, 3)


def test_parallel_host_copies_cover_every_byte(paes, gpu, orc, tmp_path):
    """Host copies split over T threads in 4 KiB-aligned parts: a length
    n = T * 4096 * m + r (0 < r < T) once lost its last r bytes, because the
    part size was rounded from floor(n / T).  Pageable lengths of that form
    for the staged ring's copy teams (T = 8 on a 16-core box), and a file
    whose last piece has that form for the file path's parallel I/O
    (L = 6n + 75 gives 6 pieces of round16(n) .. n bytes, T = 2 parts)."""
    key = bytes(range(16))
    rnd = random.Random(4096)
    for m in (160, 200, 300):  # > the 4 MiB bounce path; 4 MiB pieces, then a last piece of that form too
        for r in (1, 5, 7):
            n = 8 * 4096 * m + r
            data = np.frombuffer(rnd.randbytes(n), dtype=np.uint8)
            dst = np.zeros(n + 48, dtype=np.uint8)
            k = _run(paes, 0, data.ctypes.data, n, True, key, dst.ctypes.data)
            assert dst[:k].tobytes() == orc.encrypt_chunk(data.tobytes(), True, key), n
            back = np.zeros(n + 48, dtype=np.uint8)
            assert _run(paes, 1, dst.ctypes.data, k, True, key, back.ctypes.data) == n
            assert back[:n].tobytes() == data.tobytes(), n
    n_last = 2 * 4096 * 600 + 1
    L = 6 * n_last + 75
    data = rnd.randbytes(L)
    (tmp_path / "p.bin").write_bytes(data)
    paes.encrypt_file(str(tmp_path / "p.bin"), str(tmp_path / "c.bin"), key, workers=1)
    assert (tmp_path / "c.bin").read_bytes() == orc.encrypt_chunk(data, True, key)
    paes.decrypt_file(str(tmp_path / "c.bin"), str(tmp_path / "d.bin"), key, workers=1)
    assert (tmp_path / "d.bin").read_bytes() == data


def test_staged_ring_large_pageable_matches_device_path(paes, gpu):
    """The two-team staged ring over many 64 MiB pieces (pageable numpy
    buffers, out of place and in place) against the device-resident path on
    the same bytes, plus the decrypt round trip."""
    import torch

    key = bytes(range(3, 19))
    rk = paes.round_keys(key)
    for n in ((1 << 30) + 7, (192 << 20) + 3):
        g = torch.Generator().manual_seed(n)
        t = torch.randint(0, 256, (n,), dtype=torch.uint8, generator=g)
        src = t.numpy()
        m = (n // 16 + 1) * 16
        d_in = t.cuda()
        d_out = torch.empty(m + 16, dtype=torch.uint8, device="cuda")
        assert paes.chunk_device(0, d_in.data_ptr(), n, True, rk, d_out.data_ptr()) == m
        want = d_out[:m].cpu().numpy()
        dst = np.zeros(m + 16, dtype=np.uint8)
        assert _run(paes, 0, src.ctypes.data, n, True, key, dst.ctypes.data) == m
        assert np.array_equal(dst[:m], want), n
        inplace = np.zeros(m + 16, dtype=np.uint8)
        inplace[:n] = src
        assert _run(paes, 0, inplace.ctypes.data, n, True, key, inplace.ctypes.data) == m
        assert np.array_equal(inplace[:m], want), n
        assert _run(paes, 1, inplace.ctypes.data, m, True, key, inplace.ctypes.data) == n
        assert np.array_equal(inplace[:n], src), n


@pytest.mark.parametrize("writer", [None, "mmap", "pwrite", "mmap_space_taken_after_the_check"])
def test_run_job_on_a_full_tmpfs_is_ioerror_without_partial_output(paes, gpu, tmp_path, writer, monkeypatch):
    """An output tmpfs too small for the result: IoError (OSError), no SIGBUS
    from the shared-mapping writer, and no <out>.part.<pid> left behind
    (AtomicOutput, exec.cpp:80-106).  The last case skips the free-space check
    (as if the space went away after it): the output is mapped, the Prealloc
    thread's fallocate fails with ENOSPC and the writers report it instead of
    storing into pages that cannot be backed."""
    import subprocess

    mnt = tmp_path / "small_tmpfs"
    mnt.mkdir()
    if subprocess.run(["mount", "-t", "tmpfs", "-o", "size=1m", "tmpfs", str(mnt)], capture_output=True).returncode:
        pytest.skip("cannot mount a tmpfs here")
    try:
        if writer == "mmap_space_taken_after_the_check":
            monkeypatch.setenv("PAES_FILE_WRITER", "mmap")
            monkeypatch.setenv("PAES_FILE_SKIP_SPACE_CHECK", "1")
        elif writer:
            monkeypatch.setenv("PAES_FILE_WRITER", writer)
        src = tmp_path / "in.bin"
        src.write_bytes(os.urandom(4 << 20))
        with pytest.raises(OSError) as ei:
            paes.encrypt_file(str(src), str(mnt / "out.bin"), bytes(16), strategy="gpu")
        assert isinstance(ei.value, paes.IoError), ei.value
        assert os.listdir(mnt) == []
        # the engine is still usable: a job that fits goes through
        monkeypatch.delenv("PAES_FILE_SKIP_SPACE_CHECK", raising=False)
        small = tmp_path / "small.bin"
        small.write_bytes(os.urandom(100_000))
        assert paes.encrypt_file(str(small), str(mnt / "ok.bin"), bytes(16))["bytes_out"] == 100_000 // 16 * 16 + 16
        assert os.listdir(mnt) == ["ok.bin"]
    finally:
        subprocess.run(["umount", str(mnt)], capture_output=True)


def test_short_calls_stay_on_one_listed_gpu(paes, gpu, orc):
    """With three devices listed and ngpus = 0, a 1 KiB call is one shard, one
    launch (the size floor); 40 MiB shards three ways and still matches the
    oracle (the shard threads are the persistent pool's)."""
    rnd = random.Random(77)
    key = rnd.randbytes(16)
    paes.set_devices([0, 0, 0])
    try:
        small = rnd.randbytes(1024)
        before = paes.launch_count()
        ct = paes.encrypt_bytes(small, key)
        assert paes.launch_count() - before == 1
        assert ct == orc.encrypt_chunk(small, True, key)
        big = rnd.randbytes((40 << 20) + 5)
        for _ in range(3):  # pool threads are reused across calls
            ct = paes.encrypt_chunk(big, True, key)
            assert ct == orc.encrypt_chunk(big, True, key, threads=4)
            assert paes.decrypt_chunk(ct, True, key) == big
    finally:
        paes.set_devices([])


def test_pageable_bounce_pieces(paes, gpu, orc):
    """Pageable ranges up to 4 MiB go through a lane's two mapped bounce
    halves in balanced pieces of at most 512 KiB (runtime.cu run_bounce):
    piece edges, the 7-byte tail, exact aliasing and a wrong key, vs the oracle."""
    rnd = random.Random(512)
    key = rnd.randbytes(16)
    bad = bytes([key[0] ^ 1]) + key[1:]
    K = 512 * 1024
    for n in (0, 15, 16, K - 1, K, K + 7, 2 * K - 16, 2 * K + 1, (1 << 20) + 7, 3 * MiB + 9, 4 * MiB - 16, 4 * MiB):
        data = rnd.randbytes(n)
        src = np.frombuffer(bytearray(data) + bytearray(32), dtype=np.uint8)
        dst = np.zeros(n + 32, dtype=np.uint8)
        want = orc.encrypt_chunk(data, True, key)
        m = _run(paes, 0, src.ctypes.data, n, True, key, dst.ctypes.data)
        assert m == len(want) and dst[:m].tobytes() == want, n
        back = np.zeros(n + 32, dtype=np.uint8)
        assert _run(paes, 1, dst.ctypes.data, m, True, key, back.ctypes.data) == n
        assert back[:n].tobytes() == data, n
        # in place (exact aliasing), both directions
        buf = np.frombuffer(bytearray(want) + bytearray(16), dtype=np.uint8)
        assert _run(paes, 1, buf.ctypes.data, m, True, key, buf.ctypes.data) == n
        assert buf[:n].tobytes() == data, n
        try:
            expect = orc.decrypt_chunk(want, True, bad)
        except ValueError:
            expect = None
        if expect is None:
            _run(paes, 1, dst.ctypes.data, m, True, bad, back.ctypes.data, expect_rc=-74)
        else:
            k = _run(paes, 1, dst.ctypes.data, m, True, bad, back.ctypes.data)
            assert back[:k].tobytes() == expect


def test_device_pointer_to_a_host_entry_is_einval(paes, gpu):
    """A device buffer handed to a host-pointer entry is rejected up front
    (EINVAL, naming the buffer) instead of being dereferenced by the host."""
    import torch

    from paper_1403_7295_b200 import _native as N

    key = bytes(range(16))
    d = torch.zeros(1 << 20, dtype=torch.uint8, device="cuda")
    h = np.zeros((1 << 20) + 16, dtype=np.uint8)
    L = N.load()
    olen = C.c_uint64()
    for src, dst, which in ((d.data_ptr(), h.ctypes.data, "input"), (h.ctypes.data, d.data_ptr(), "output")):
        for n in (4096, 8 << 20):  # the lane path and the ring path
            rc = L.paes_cuda_chunk(0, src, n, 1, paes.round_keys(key), dst, C.byref(olen), 1)
            assert rc == N.EINVAL and which in N.last_error() and "device memory" in N.last_error()
    # the library still works afterwards
    data = os.urandom(5000)
    assert paes.decrypt_bytes(paes.encrypt_bytes(data, key), key) == data
