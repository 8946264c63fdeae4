"""Device-pointer transforms inside CUDA graphs: an encrypt (and an unchecked
decrypt) launched through the C ABI on a capturing stream is recorded as a
graph node and replays bit-exactly -- callers can fold the hot path into
their own graphs instead of paying a launch per call."""
import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_chunk_device_captures_and_replays(paes, gpu, orc):
    import torch

    rnd = random.Random(9)
    key = rnd.randbytes(16)
    rk = paes.round_keys(key)
    n = 3 * 1024 * 1024 + 5
    src = torch.zeros(n + 64, dtype=torch.uint8, device="cuda")
    ct = torch.zeros(n + 64, dtype=torch.uint8, device="cuda")
    pt = torch.zeros(n + 64, dtype=torch.uint8, device="cuda")
    base = paes.launch_count()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        # warm the device context outside the capture
        paes.chunk_device(paes.ENCRYPT, src.data_ptr(), n, True, rk, ct.data_ptr(), 0, s.cuda_stream)
        s.synchronize()
        with torch.cuda.graph(g, stream=s):
            m = paes.chunk_device(paes.ENCRYPT, src.data_ptr(), n, True, rk, ct.data_ptr(), 0, s.cuda_stream)
            # non-final decrypt: no trailer check, so no host sync inside the capture
            paes.chunk_device(paes.DECRYPT, ct.data_ptr(), m, False, rk, pt.data_ptr(), 0, s.cuda_stream)
    assert m == (n // 16 + 1) * 16
    for rep in range(3):
        data = rnd.randbytes(n)
        src[:n].copy_(torch.frombuffer(bytearray(data), dtype=torch.uint8))
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        assert ct[:m].cpu().numpy().tobytes() == orc.encrypt_chunk(data, True, key), rep
        assert pt[:n].cpu().numpy().tobytes() == data, rep
    # the library counts launches at capture time, not at replay
    assert paes.launch_count() - base == 3


def test_batch_plan_captures_and_replays(paes, gpu, orc):
    import torch

    rnd = random.Random(10)
    lens = [rnd.randrange(0, 70_000) for _ in range(23)]
    keys = [rnd.randbytes(16) for _ in lens]
    in_off, out_off, oi, oo = [], [], 0, 0
    for L in lens:
        in_off.append(oi)
        out_off.append(oo)
        oi += (L + 15) // 16 * 16
        oo += (L // 16 + 1) * 16
    rks = b"".join(paes.round_keys(k) for k in keys)
    src = torch.zeros(oi + 16, dtype=torch.uint8, device="cuda")
    dst = torch.zeros(oo + 16, dtype=torch.uint8, device="cuda")
    plan = paes.BatchPlan(paes.ENCRYPT, in_off, out_off, lens, rks, True)
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    try:
        with torch.cuda.stream(s):
            plan.run(src.data_ptr(), dst.data_ptr(), s.cuda_stream)
            s.synchronize()
            with torch.cuda.graph(g, stream=s):
                plan.run(src.data_ptr(), dst.data_ptr(), s.cuda_stream)
        for rep in range(2):
            msgs = [rnd.randbytes(L) for L in lens]
            h = np.zeros(oi + 16, dtype=np.uint8)
            for o, m in zip(in_off, msgs):
                h[o:o + len(m)] = np.frombuffer(m, dtype=np.uint8)
            src.copy_(torch.from_numpy(h))
            torch.cuda.synchronize()
            g.replay()
            torch.cuda.synchronize()
            out = dst.cpu().numpy()
            for o, m, k in zip(out_off, msgs, keys):
                want = orc.encrypt_chunk(m, True, k)
                assert out[o:o + len(want)].tobytes() == want, rep
    finally:
        plan.close()


def test_final_decrypt_async_captures_and_replays(paes, gpu, orc):
    """The queued final decrypt (paes_cuda_chunk_device_async) records into a
    graph with the encrypt before it; each replay re-checks the trailer and
    writes the unpadded length -- or BAD_PAD under a wrong key -- on the device."""
    import torch

    rnd = random.Random(11)
    key = rnd.randbytes(16)
    rk, bad = paes.round_keys(key), paes.round_keys(bytes(16))
    n = 2 * 1024 * 1024 + 9
    m = (n // 16 + 1) * 16
    src = torch.zeros(n + 64, dtype=torch.uint8, device="cuda")
    ct = torch.zeros(m + 64, dtype=torch.uint8, device="cuda")
    pt = torch.zeros(m + 64, dtype=torch.uint8, device="cuda")
    res = torch.zeros(3, dtype=torch.int64, device="cuda")
    s = torch.cuda.Stream()
    base = paes.launch_count()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        paes.chunk_device_async(paes.ENCRYPT, src.data_ptr(), n, True, rk, ct.data_ptr(), res.data_ptr(), 0,
                                s.cuda_stream)
        s.synchronize()
        with torch.cuda.graph(g, stream=s):
            paes.chunk_device_async(paes.ENCRYPT, src.data_ptr(), n, True, rk, ct.data_ptr(), res.data_ptr(), 0,
                                    s.cuda_stream)
            paes.chunk_device_async(paes.DECRYPT, ct.data_ptr(), m, True, rk, pt.data_ptr(), res.data_ptr() + 8, 0,
                                    s.cuda_stream)
            paes.chunk_device_async(paes.DECRYPT, ct.data_ptr(), m, True, bad, pt.data_ptr() + 0, res.data_ptr() + 16,
                                    0, s.cuda_stream)
    assert paes.launch_count() - base == 4
    for rep in range(3):
        data = rnd.randbytes(n)
        src[:n].copy_(torch.frombuffer(bytearray(data), dtype=torch.uint8))
        res.fill_(-2)
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        got = [int(x) & ((1 << 64) - 1) for x in res.cpu().tolist()]
        assert got[0] == m and got[1] == n, (rep, got)
        want_ct = orc.encrypt_chunk(data, True, key)
        assert ct[:m].cpu().numpy().tobytes() == want_ct, rep
        # the wrong key's verdict is whatever unpad_final says of its last block
        u = orc.unpad(orc.ecb(1, want_ct[-16:], bytes(16)))  # unpadded length of the last block, or < 0
        assert got[2] == (paes.BAD_PAD if u < 0 else m - 16 + u), (rep, got, u)


def test_async_result_word_in_mapped_memory_and_empty_inputs(paes, gpu):
    """d_result may be mapped pinned host memory; empty transforms still write
    their result (0) in stream order, and a final encrypt of 0 bytes writes the
    full pad block (16)."""
    import torch

    rk = paes.round_keys(bytes(range(16)))
    host = torch.full((4,), -2, dtype=torch.int64).pin_memory()
    # torch's pinned blocks are cudaHostAlloc'ed: mapped at the same address under UVA
    ct = torch.zeros(64, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    hp = host.data_ptr()
    paes.chunk_device_async(paes.ENCRYPT, ct.data_ptr(), 0, True, rk, ct.data_ptr(), hp, 0, s.cuda_stream)
    paes.chunk_device_async(paes.ENCRYPT, ct.data_ptr(), 0, False, rk, ct.data_ptr(), hp + 8, 0, s.cuda_stream)
    paes.chunk_device_async(paes.DECRYPT, ct.data_ptr(), 16, True, rk, ct.data_ptr() + 16, hp + 16, 0, s.cuda_stream)
    s.synchronize()
    assert host.tolist()[:3] == [16, 0, 0]  # E(16 x 0x10) decrypts back to an all-pad block: unpadded length 0
    with pytest.raises(paes.PaddingError):
        paes.chunk_device_async(paes.DECRYPT, ct.data_ptr(), 0, True, rk, ct.data_ptr(), hp, 0, s.cuda_stream)
    with pytest.raises(ValueError):
        paes.chunk_device_async(paes.ENCRYPT, ct.data_ptr(), 16, True, rk, ct.data_ptr(), hp + 4, 0, s.cuda_stream)


def test_batch_plan_run_async_lengths_and_bad_trailers(paes, gpu, orc):
    """Queued batch decrypt: per-message unpadded lengths land in a device
    array, malformed trailers (wrong keys) as BAD_PAD at exactly those
    messages, empty messages as 0; the run replays from a CUDA graph."""
    import torch

    rnd = random.Random(12)
    lens = [rnd.randrange(0, 50_000) for _ in range(40)]
    keys = [rnd.randbytes(16) for _ in lens]
    msgs = [rnd.randbytes(L) for L in lens]
    cts = [orc.encrypt_chunk(m, True, k) for m, k in zip(msgs, keys)]
    bad = {3, 17, 29}
    rks = b"".join(paes.round_keys(bytes(16) if i in bad else k) for i, k in enumerate(keys))
    off, o = [], 0
    for c in cts:
        off.append(o)
        o += len(c)
    src = torch.frombuffer(bytearray(b"".join(cts)), dtype=torch.uint8).cuda()
    dst = torch.zeros(o + 16, dtype=torch.uint8, device="cuda")
    res = torch.full((len(lens),), -7, dtype=torch.int64, device="cuda")
    plan = paes.BatchPlan(paes.DECRYPT, off, off, [len(c) for c in cts], rks, True)
    try:
        s = torch.cuda.Stream()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            plan.run_async(src.data_ptr(), dst.data_ptr(), res.data_ptr(), s.cuda_stream)
            s.synchronize()
            with torch.cuda.graph(g, stream=s):
                plan.run_async(src.data_ptr(), dst.data_ptr(), res.data_ptr(), s.cuda_stream)
        for rep in range(2):
            res.fill_(-7)
            torch.cuda.synchronize()
            g.replay()
            torch.cuda.synchronize()
            got = [int(x) & ((1 << 64) - 1) for x in res.tolist()]
            out = dst.cpu().numpy().tobytes()
            for i, (m, c) in enumerate(zip(msgs, cts)):
                if i in bad:
                    u = orc.unpad(orc.ecb(1, c[-16:], bytes(16)))
                    assert got[i] == (paes.BAD_PAD if u < 0 else len(c) - 16 + u), (rep, i)
                else:
                    assert got[i] == len(m), (rep, i)
                    assert out[off[i]:off[i] + len(m)] == m, (rep, i)
    finally:
        plan.close()
    # an encrypt plan with an empty, unpadded message: its length is 0
    enc = paes.BatchPlan(paes.ENCRYPT, [0, 0], [0, 32], [0, 32], rks[:352], False)
    try:
        r2 = torch.full((2,), -7, dtype=torch.int64, device="cuda")
        enc.run_async(src.data_ptr(), dst.data_ptr(), r2.data_ptr())
        torch.cuda.synchronize()
        assert r2.tolist() == [0, 32]
    finally:
        enc.close()
