"""The bitsliced (LOP3) encrypt kernel of the T-table vs bitsliced A/B
(scripts/bitsliced_ab.py) must produce the same bytes as the reference."""
import ctypes as C
import os

import pytest

pytestmark = pytest.mark.gpu


def test_bitsliced_matches_oracle(paes, gpu, orc):
    import torch

    from paper_1403_7295_b200 import build as B

    fn = C.CDLL(B.BITSLICED_AB).paes_bitsliced_ab_ecb
    fn.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p]
    key = os.urandom(16)
    data = os.urandom(16 * 1024 * 37)
    src = torch.frombuffer(bytearray(data), dtype=torch.uint8).cuda()
    dst = torch.empty_like(src)
    assert fn(src.data_ptr(), dst.data_ptr(), len(data), paes.round_keys(key), None) == 0
    torch.cuda.synchronize()
    assert dst.cpu().numpy().tobytes() == orc.ecb(0, data, key, threads=4)
    assert fn(src.data_ptr(), dst.data_ptr(), 100, paes.round_keys(key), None) == -22
