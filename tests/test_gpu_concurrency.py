"""Concurrent calls from many host threads (the reference runs encrypt_ecb
from W threads at once, exec.cpp:153-175): every API path must stay
bit-exact when its calls interleave.  ctypes releases the GIL, so the
threads really run inside the library together."""
import os
import random
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_concurrent_mixed_calls(paes, gpu, orc):
    import torch

    rnd = random.Random(99)
    jobs = []
    for i in range(48):
        kind = ["bytes", "ecb", "device", "batch", "pageable_big"][i % 5]
        n = rnd.choice([0, 1, 17, 1000, 65536, 300_001, 3 << 20])
        jobs.append((kind, n, os.urandom(16), os.urandom(n)))

    def run(job):
        kind, n, key, data = job
        if kind == "bytes":
            ct = paes.encrypt_bytes(data, key)
            assert ct == orc.encrypt_chunk(data, True, key)
            assert paes.decrypt_bytes(ct, key) == data
        elif kind == "ecb":
            d = data[: len(data) - len(data) % 16]
            assert paes.encrypt_ecb(d, key) == orc.ecb(0, d, key)
        elif kind == "device":
            s = torch.cuda.Stream()
            src = torch.frombuffer(bytearray(data + b"\0" * 16), dtype=torch.uint8).cuda()
            dst = torch.zeros(len(data) + 32, dtype=torch.uint8, device="cuda")
            torch.cuda.synchronize()
            m = paes.chunk_device(0, src.data_ptr(), n, True, paes.round_keys(key), dst.data_ptr(), 0, s.cuda_stream)
            s.synchronize()
            assert dst[:m].cpu().numpy().tobytes() == orc.encrypt_chunk(data, True, key)
        elif kind == "batch":
            parts = [data[:n // 3], data[n // 3:]]
            keys = [key, bytes(reversed(key))]
            in_off = [0, (len(parts[0]) + 15) // 16 * 16]
            total_in = in_off[1] + len(parts[1]) + 16
            out_off = [0, (len(parts[0]) // 16 + 1) * 16]
            total_out = out_off[1] + (len(parts[1]) // 16 + 1) * 16
            hin = np.zeros(total_in, dtype=np.uint8)
            hin[in_off[0]:in_off[0] + len(parts[0])] = np.frombuffer(parts[0], dtype=np.uint8)
            hin[in_off[1]:in_off[1] + len(parts[1])] = np.frombuffer(parts[1], dtype=np.uint8)
            hout = np.zeros(total_out, dtype=np.uint8)
            rks = b"".join(paes.round_keys(k) for k in keys)
            ol = paes.ecb_batch_host(0, hin.ctypes.data, hout.ctypes.data, in_off, out_off,
                                     [len(p) for p in parts], rks, True)
            for i in range(2):
                assert hout[out_off[i]:out_off[i] + ol[i]].tobytes() == orc.encrypt_chunk(parts[i], True, keys[i])
        else:  # pageable, several pieces through the staged ring
            big = data * 4
            assert paes.encrypt_bytes(big, key) == orc.encrypt_chunk(big, True, key, threads=2)
        return kind

    with ThreadPoolExecutor(12) as ex:
        done = list(ex.map(run, jobs))
    assert len(done) == len(jobs)


def test_one_checked_plan_from_many_threads(paes, gpu, orc):
    """A decrypt plan with trailer checks run concurrently on several streams:
    the shared status words are serialised, every run sees its own lengths."""
    import torch

    rnd = random.Random(5)
    lens = [rnd.randrange(0, 40_000) for _ in range(37)]
    keys = [rnd.randbytes(16) for _ in lens]
    msgs = [rnd.randbytes(n) for n in lens]
    cts = [orc.encrypt_chunk(m, True, k) for m, k in zip(msgs, keys)]
    offs, o = [], 0
    for c in cts:
        offs.append(o)
        o += len(c)
    src = torch.from_numpy(np.frombuffer(b"".join(cts), dtype=np.uint8).copy()).cuda()
    rks = b"".join(paes.round_keys(k) for k in keys)
    plan = paes.BatchPlan(paes.DECRYPT, offs, offs, [len(c) for c in cts], rks, True)

    def worker(t):
        stream = torch.cuda.Stream()
        dst = torch.zeros(o, dtype=torch.uint8, device="cuda")
        for _ in range(10):
            with torch.cuda.stream(stream):
                got = plan.run(src.data_ptr(), dst.data_ptr(), stream.cuda_stream)
            assert got == lens, t
        stream.synchronize()
        h = dst.cpu().numpy()
        return all(h[off:off + n].tobytes() == m for off, n, m in zip(offs, lens, msgs))

    try:
        with ThreadPoolExecutor(4) as ex:
            assert all(ex.map(worker, range(4)))
    finally:
        plan.close()


def test_concurrent_final_device_decrypts_keep_their_own_verdicts(paes, gpu, orc):
    """Final device-pointer decrypts on private streams from many threads at
    once, valid and wrong keys mixed: every call reads its own trailer status
    (per-call status slots), never a neighbour's."""
    import torch

    rnd = random.Random(88)
    jobs = []
    for t in range(12):
        key = rnd.randbytes(16)
        data = rnd.randbytes(rnd.choice([16, 4096 + 3, 3 << 20]))
        ct = orc.encrypt_chunk(data, True, key)
        bad = t % 3 == 0
        use_key = bytes([key[0] ^ 0x5A]) + key[1:] if bad else key
        if bad:  # keep only wrong keys whose trailer is certainly invalid
            try:
                orc.decrypt_chunk(ct, True, use_key)
                bad = False
                use_key = key
            except ValueError:
                pass
        jobs.append((data, ct, use_key, bad))

    def run(job):
        data, ct, key, bad = job
        s = torch.cuda.Stream()
        src = torch.frombuffer(bytearray(ct), dtype=torch.uint8).to("cuda")
        dst = torch.zeros(len(ct), dtype=torch.uint8, device="cuda")
        torch.cuda.synchronize()
        ok = True
        for _ in range(5):
            try:
                n = paes.chunk_device(1, src.data_ptr(), len(ct), True, paes.round_keys(key), dst.data_ptr(), 0,
                                      s.cuda_stream)
                ok &= (not bad) and n == len(data) and dst[:n].cpu().numpy().tobytes() == data
            except paes.PaddingError:
                ok &= bad
        return ok

    with ThreadPoolExecutor(12) as ex:
        assert all(ex.map(run, jobs))


def test_short_calls_from_many_threads_share_lanes_exactly(paes, gpu, orc):
    """Short host calls (pinned zero-copy up to the zero-copy limit, pageable
    bounce up to 4 MiB) run on leased lanes without the device lock
    (runtime.cu run_short): 16 threads x 40 calls of mixed sizes, pinned and
    pageable, encrypt and final decrypt, 1 in 8 decrypts with a wrong key.
    Every result is the oracle's, every wrong key is PaddingError, and no
    thread sees another's verdict or bytes."""
    import ctypes as C

    import torch

    from paper_1403_7295_b200 import _native as N

    L = N.load()
    sizes = [0, 5, 16, 4095, 4096, 65543, 1 << 20]

    def worker(t):
        rnd = random.Random(1000 + t)
        hin = torch.empty((1 << 20) + 32, dtype=torch.uint8).pin_memory()
        hout = torch.empty((1 << 20) + 32, dtype=torch.uint8).pin_memory()
        for i in range(40):
            n = rnd.choice(sizes)
            key = os.urandom(16)
            data = os.urandom(n)
            want = orc.encrypt_chunk(data, True, key)
            if rnd.random() < 0.5:  # pinned: zero-copy kernel on the caller's buffers
                hin[:n] = torch.frombuffer(bytearray(data), dtype=torch.uint8) if n else hin[:0]
                ol = C.c_uint64(0)
                rc = L.paes_cuda_chunk(0, C.c_void_p(hin.data_ptr()), n, 1, paes.round_keys(key),
                                       C.c_void_p(hout.data_ptr()), C.byref(ol), 1)
                assert rc == 0 and ol.value == len(want)
                ct = hout[:ol.value].numpy().tobytes()
                assert ct == want, (t, i, n, "pinned enc")
                hin[:len(ct)] = torch.frombuffer(bytearray(ct), dtype=torch.uint8)
                bad = rnd.random() < 0.125
                rc = L.paes_cuda_chunk(1, C.c_void_p(hin.data_ptr()), len(ct), 1,
                                       paes.round_keys(bytes(16) if bad else key), C.c_void_p(hout.data_ptr()),
                                       C.byref(ol), 1)
                if bad:
                    assert rc == N.EBADMSG or (rc == 0 and hout[:ol.value].numpy().tobytes() != data)
                else:
                    assert rc == 0 and hout[:ol.value].numpy().tobytes() == data, (t, i, n, "pinned dec")
            else:  # pageable: the lane's bounce buffer
                ct = paes.encrypt_bytes(data, key)
                assert ct == want, (t, i, n, "pageable enc")
                if rnd.random() < 0.125:
                    try:
                        out = paes.decrypt_bytes(ct, bytes(16))
                        assert out != data
                    except paes.PaddingError:
                        pass
                else:
                    assert paes.decrypt_bytes(ct, key) == data, (t, i, n, "pageable dec")
        return t

    with ThreadPoolExecutor(16) as ex:
        assert sorted(ex.map(worker, range(16))) == list(range(16))


def test_more_short_callers_than_lanes_wait_their_turn(paes, gpu, orc):
    """96 threads at once against a pool capped at 64 lanes per device: the
    extra callers wait for a lane instead of failing or deadlocking."""
    key = bytes(range(16))
    data = [os.urandom(4096 + i) for i in range(96)]

    def run(i):
        for _ in range(5):
            ct = paes.encrypt_bytes(data[i], key)
            assert paes.decrypt_bytes(ct, key) == data[i]
        return ct

    with ThreadPoolExecutor(96) as ex:
        cts = list(ex.map(run, range(96)))
    for i in (0, 47, 95):
        assert cts[i] == orc.encrypt_chunk(data[i], True, key)
