"""The reference's single-state API (aes.hpp:72-78, aes.cpp:194-227) run on
the GPU, bit-exact against the oracle's restatement on random states, plus
the known answers of test_aes.cpp:136-253."""
import random

import pytest

pytestmark = pytest.mark.gpu


def test_all_ops_vs_oracle(paes, gpu, orc):
    rnd = random.Random(2020)
    n = 20000  # test_aes.cpp:228-237 runs 20000 random MixColumns round trips
    states = rnd.randbytes(16 * n)
    rk = rnd.randbytes(16)
    for op in range(7):
        got = paes.state_transform(op, states, rk if op == paes.ADD_ROUND_KEY else None)
        want = b"".join(orc.transform(op, states[16 * i:16 * i + 16], rk) for i in range(n))
        assert got == want, op  # every one of the 20000 states
    # inverses round-trip every state
    for fwd, inv in ((paes.SUB_BYTES, paes.INV_SUB_BYTES), (paes.SHIFT_ROWS, paes.INV_SHIFT_ROWS),
                     (paes.MIX_COLUMNS, paes.INV_MIX_COLUMNS)):
        assert paes.state_transform(inv, paes.state_transform(fwd, states)) == states


def test_known_answers(paes, gpu):
    col = bytes([0xDB, 0x13, 0x53, 0x45]) + bytes(12)
    assert paes.state_transform(paes.MIX_COLUMNS, col)[:4].hex() == "8e4da1bc"
    ones = bytes([1] * 16)
    assert paes.state_transform(paes.MIX_COLUMNS, ones) == ones
    sb = paes.sbox()
    assert paes.state_transform(paes.SUB_BYTES, bytes(range(256))) == sb
    assert paes.state_transform(paes.INV_SUB_BYTES, sb) == bytes(range(256))
