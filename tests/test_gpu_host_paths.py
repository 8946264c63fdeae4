"""The three host-pointer paths of paes_cuda_chunk, each forced explicitly:
zero-copy small ranges, the pinned direct ring, and the staged ring for
pageable memory -- all bit-exact vs the oracle across piece boundaries."""
import ctypes as C
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
MiB = 1 << 20


def _run(paes, direction, src_ptr, n, final, key, dst_ptr):
    from paper_1403_7295_b200 import _native as N

    olen = C.c_uint64()
    rc = N.load().paes_cuda_chunk(direction, src_ptr, n, int(final), paes.round_keys(key), dst_ptr, C.byref(olen), 1)
    assert rc == 0, N.last_error()
    return olen.value


@pytest.mark.parametrize("pinned", [True, False])
def test_ring_paths_vs_oracle(paes, gpu, orc, pinned):
    import torch

    paes.set_pipeline(64 * 1024, 3)  # tiny pieces: many slots in flight, small-path threshold 64 KiB
    try:
        key = os.urandom(16)
        for n in [100, 64 * 1024, 64 * 1024 + 1, 3 * 64 * 1024 + 7, 1_000_003]:
            data = os.urandom(n)
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
    finally:
        paes.set_pipeline(64 * MiB, 3)
