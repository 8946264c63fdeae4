"""Pin the oracle (oracle/aes_oracle.c) before trusting it: reference KATs
(test_aes.cpp), the survey's golden SHA-256 digests, vectors
produced by the reference's own _paes module (tests/golden/golden.json), and
bit-equality with the reference compiled from its sources (oracle/_ref)."""
from __future__ import annotations

import hashlib
import os
import random

import pytest

KEY_C1 = bytes.fromhex("000102030405060708090a0b0c0d0e0f")


def test_fips_vectors(orc):
    """test_aes.cpp:255-269, test_smoke.py:14-18."""
    assert orc.encrypt_block(bytes.fromhex("3243f6a8885a308d313198a2e0370734"),
                             bytes.fromhex("2b7e151628aed2a6abf7158809cf4f3c")).hex() == \
        "3925841d02dc09fbdc118597196a0b32"
    ct = orc.encrypt_block(bytes.fromhex("00112233445566778899aabbccddeeff"), KEY_C1)
    assert ct.hex() == "69c4e0d86a7b0430d8cdb78070b4c55a"
    assert orc.decrypt_block(ct, KEY_C1).hex() == "00112233445566778899aabbccddeeff"


def test_zero_key_snapshot(orc):
    """test_aes.cpp:285-292."""
    assert orc.decrypt_block(bytes(16), bytes(16)).hex() == "140f0f1011b5223d79587717ffd9ec3a"


def _gf_mul_oracle(a, b):
    """Independent carry-less multiply + long division (test_aes.cpp:19-28)."""
    acc = 0
    for i in range(8):
        if b & (1 << i):
            acc ^= a << i
    for bit in range(15, 7, -1):
        if acc & (1 << bit):
            acc ^= 0x11B << (bit - 8)
    return acc


def _sbox_entry(a):
    inv = 0 if a == 0 else next(b for b in range(1, 256) if _gf_mul_oracle(a, b) == 1)
    out = 0
    for i in range(8):
        bit = ((inv >> i) ^ (inv >> ((i + 4) % 8)) ^ (inv >> ((i + 5) % 8)) ^ (inv >> ((i + 6) % 8)) ^
               (inv >> ((i + 7) % 8)) ^ (0x63 >> i)) & 1
        out |= bit << i
    return out


def test_sbox_against_gf_oracle(orc):
    """test_aes.cpp:79-96."""
    s, si = orc.sbox(), orc.inv_sbox()
    assert s[0x00] == 0x63 and s[0x53] == 0xED
    for i in range(256):
        assert s[i] == _sbox_entry(i)
        assert si[s[i]] == i


def test_gf_mul(orc):
    rnd = random.Random(7)
    for _ in range(2000):
        a, b = rnd.randrange(256), rnd.randrange(256)
        assert orc.L.oracle_gf_mul(a, b) == _gf_mul_oracle(a, b)


def test_key_schedule_kats(orc, golden):
    """test_aes.cpp:107-134 + schedules from the reference _paes.expand_key."""
    assert orc.expand_key(bytes(16))[16:32].hex() == "62636363" * 4
    assert orc.expand_key(bytes.fromhex("2b7e151628aed2a6abf7158809cf4f3c"))[16:20].hex() == "a0fafe17"
    for e in golden["key_schedules"]:
        assert orc.expand_key(bytes.fromhex(e["key"])).hex() == e["rk"]


def test_round_transforms(orc):
    """test_aes.cpp:147-253: mix_columns column vector, shift_rows, inverses."""
    st = bytearray(16)
    st[0:4] = bytes([0xDB, 0x13, 0x53, 0x45])
    assert orc.transform(4, bytes(st))[0:4].hex() == "8e4da1bc"
    assert orc.transform(4, bytes([1] * 4 + [0] * 12))[0:4] == bytes([1] * 4)
    rnd = random.Random(13)
    for _ in range(500):
        s = bytes(rnd.randrange(256) for _ in range(16))
        assert orc.transform(5, orc.transform(4, s)) == s
        assert orc.transform(3, orc.transform(2, s)) == s
        assert orc.transform(1, orc.transform(0, s)) == s
        x = s
        for _ in range(4):
            x = orc.transform(2, x)
        assert x == s
    row1 = bytearray(16)
    row1[1], row1[5], row1[9], row1[13] = b"abcd"
    sh = orc.transform(2, bytes(row1))
    assert (sh[1], sh[5], sh[9], sh[13]) == tuple(b"bcda")


def test_golden_bytes(orc, golden):
    for e in golden["bytes"]:
        key, pt = bytes.fromhex(e["key"]), bytes.fromhex(e["pt"])
        ct = orc.encrypt_chunk(pt, True, key)
        if "ct" in e:
            assert ct.hex() == e["ct"]
        else:
            assert hashlib.sha256(ct).hexdigest() == e["ct_sha256"]
        assert orc.decrypt_chunk(ct, True, key) == pt


def test_golden_pad_unpad_plans(orc, golden):
    for e in golden["pad"]:
        data = bytes.fromhex(e["in"])
        out = bytearray(len(data) + 16)
        n = orc.L.oracle_pad_final((__import__("ctypes").c_uint8 * max(len(data), 1)).from_buffer_copy(data or b"\0"),
                                   len(data), (__import__("ctypes").c_uint8 * len(out)).from_buffer(out))
        assert bytes(out[:n]).hex() == e["out"]
    for e in golden["unpad"]:
        r = orc.unpad(bytes.fromhex(e["in"]))
        if e["ok"]:
            assert r == len(e["out"]) // 2
        else:
            assert r == -74
    for e in golden["plans"]:
        got = orc.plan(0, e["total"], e["workers"])
        assert [list(c) for c in got] == e["chunks"]


def test_survey_digests_cfg1_cfg3(orc):
    """sha256 of pt and ct for cfg1 (64 MiB) and cfg3 1K/64K/1M."""
    key = orc.sweep(0, 16)
    assert key.hex() == "4c287f4282c15e6cfda0c041590ebc2a"
    pt = orc.sweep(0, 64 << 20)
    assert hashlib.sha256(pt).hexdigest() == "7f42e6ca8d5dd69801932708ee58cbf3fa4f5c066a22dc792fd4e6059969325f"
    ct = orc.encrypt_chunk(pt, True, key, threads=os.cpu_count() or 4)
    assert hashlib.sha256(ct).hexdigest() == "2d8284614df3ca943d7e0ac3bedac30a15ff45797dddbaf734a3a454245b74d0"
    assert ct[:16].hex() == "917d63a1c10eb394b3960d0bfc15d2a6" and ct[-16:].hex() == "80ebbb18c31c1825f602f68fd1e87cd9"
    key2 = orc.sweep(2, 16)
    assert key2.hex() == "a2b4856de87168738bc748814df5db32"
    for L, hpt, hct in [
        (1031, "9b88a718d4c62bf8d782c159df0f24ea277aaba0704ec20b6bfd848b6109beed",
         "6ac26a3cb670d42e347ded1995365cdef5e52c6e94a375e411f65f72e6cc4cc0"),
        (65543, "2b27e9e82e0ee264e3f5a109550b12caf2249b6271550464f9fdf1d0f94ec94f",
         "47a89af02d59972ef977ace6b776cf639941dae06b704440dede8606e3ac5ef1"),
        (1048583, "d600c7601cb82813c01d372d64430e7dbb83100a8b575da4d3ae1f06736fdf44",
         "3f905b0e51b3bbaf419fb7adcc8cb3a5baa92c60f40c0f73af8ae10ff960cf24"),
    ]:
        pt = orc.sweep(2, L)
        assert hashlib.sha256(pt).hexdigest() == hpt
        ct = orc.encrypt_chunk(pt, True, key2)
        assert hashlib.sha256(ct).hexdigest() == hct
        assert ct[-16:] == orc.encrypt_block(pt[-7:] + bytes([9] * 9), key2)  # 7-byte tail + nine 0x09


def test_digests_self_consistent(orc, digests):
    """The reference-computed digests agree with the oracle where cheap."""
    assert digests["cfg1"]["ct_sha256"] == "2d8284614df3ca943d7e0ac3bedac30a15ff45797dddbaf734a3a454245b74d0"
    d3 = {e["S"]: e for e in digests["cfg3"]["sizes"]}
    key2 = orc.sweep(2, 16)
    pt = orc.sweep(2, (64 << 10) + 7)
    assert hashlib.sha256(orc.encrypt_chunk(pt, True, key2)).hexdigest() == d3[64 << 10]["ct_sha256"]
    lens = orc.batch_lengths(4, digests["cfg5"]["n"])
    assert sum(lens) == digests["cfg5"]["total_len"]
    k = orc.sweep((4 << 32) + 5, 16)
    m = orc.sweep((4 << 32) + 5, lens[5])
    assert hashlib.sha256(orc.encrypt_chunk(m, True, k)).hexdigest()[:16] == digests["cfg5"]["ct_msg_sha256_16"][5]
    d4 = digests["cfg4"]
    win = d4["window"]
    off = 0
    pt = orc.counter_fill(3, off, win)
    assert hashlib.sha256(orc.ecb(0, pt, orc.sweep(3, 16), threads=4)).hexdigest() == d4["window_sha256"]["0"]
    assert orc.encrypt_chunk(b"", True, orc.sweep(3, 16)).hex() == d4["pad_block"]


# ------------------------------------------------------------- vs the reference itself
def test_oracle_equals_reference_build(orc, ref):
    rnd = random.Random(5)
    for n in [0, 1, 15, 16, 17, 100, 1000, 4096 + 3, 100_003]:
        key = bytes(rnd.randrange(256) for _ in range(16))
        data = os.urandom(n)
        assert orc.encrypt_chunk(data, True, key) == ref.chunk(0, data, True, key)
        ct = ref.chunk(0, data, True, key)
        assert orc.decrypt_chunk(ct, True, key) == ref.chunk(1, ct, True, key) == data
        if n % 16 == 0:
            assert orc.ecb(1, data, key) == ref.ecb(1, data, key)
        assert orc.expand_key(key) == ref.expand_key(key)
    for total in range(0, 300, 7):
        for w in (1, 2, 3, 8, 33):
            assert orc.plan(0, total, w) == ref.plan(0, total, w)
            assert orc.plan(1, total, w) == ref.plan(1, total, w)
    assert orc.sweep(7, 1000) == ref.sweep(7, 1000)
    assert orc.sweep(0, 16) == ref.sweep(0, 16)


def test_plan_grid_vs_reference(orc, ref):
    """acceptance.cpp:348-384 grid (0..1024 x 1..33), sampled densely."""
    for total in range(0, 1025, 3):
        for w in range(1, 34, 4):
            assert orc.plan(0, total, w) == ref.plan(0, total, w)


def test_reject_outliers_golden(ref, golden):
    for e in golden["reject_outliers"]:
        assert ref.reject_outliers(e["in"]) == pytest.approx(e["out"])
