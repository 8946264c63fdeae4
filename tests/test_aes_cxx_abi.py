"""lib/libpaes_aes_b200.so -- the reference's aes.cpp entry points as C++ symbols
over the engine (csrc/aes_cxx_abi.cpp), the link-level drop-in.

CPU: the library exports exactly the functions the reference's aes.cpp
defines (tests/golden/aes_symbols.txt, made from the reference object by
tests/golden/make_aes_symbols.sh), resolves against libpaes_cuda.so, and its
host-side members (RoundKeySchedule's constructor = host key expansion,
north_star (1); sbox()/inv_sbox()) give the FIPS-197 values.  GPU: the bulk
and single-block entries, called through their Itanium-ABI signatures
(std::span by value = pointer + size in two registers; State by value = 16
bytes in two registers), match the oracle.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1403_7295_b200", "lib", "libpaes_aes_b200.so")
GOLDEN = os.path.join(ROOT, "tests", "golden", "aes_symbols.txt")

CTOR = "_ZN4paes3aes16RoundKeyScheduleC1ERKNS0_6Key128E"
SBOX = "_ZN4paes3aes4sboxEv"
INV_SBOX = "_ZN4paes3aes8inv_sboxEv"
ENC_ECB = "_ZN4paes3aes11encrypt_ecbESt4spanIKhLm18446744073709551615EES1_IhLm18446744073709551615EERKNS0_16RoundKeyScheduleE"
DEC_ECB = "_ZN4paes3aes11decrypt_ecbESt4spanIKhLm18446744073709551615EES1_IhLm18446744073709551615EERKNS0_16RoundKeyScheduleE"
ENC_BLOCK = "_ZN4paes3aes13encrypt_blockERKSt5arrayIhLm16EERKNS0_16RoundKeyScheduleE"
MIX = "_ZN4paes3aes11mix_columnsENS0_5StateE"
INV_MIX = "_ZN4paes3aes15inv_mix_columnsENS0_5StateE"


class State(C.Structure):
    _fields_ = [("cells", C.c_uint8 * 16)]


@pytest.fixture(scope="module")
def aeslib():
    if not os.path.exists(LIB):
        pytest.fail("lib/libpaes_aes_b200.so missing: run __graft_entry__.build()")
    from paper_1403_7295_b200 import _native

    _native.load()  # libpaes_cuda.so first (the library's DT_NEEDED, same path)
    return C.CDLL(LIB)


def _defined(path):
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True, check=True).stdout
    return {ln.split()[2] for ln in out.splitlines() if len(ln.split()) == 3 and ln.split()[1] == "T"}


def test_exports_exactly_the_reference_aes_symbols(aeslib):
    want = {ln.strip() for ln in open(GOLDEN) if ln.strip()}
    assert len(want) == 16
    assert _defined(LIB) == want


def _schedule(aeslib, key: bytes):
    ks = (C.c_uint8 * 176)()
    k = (C.c_uint8 * 16).from_buffer_copy(key)
    ctor = getattr(aeslib, CTOR)
    ctor.restype = None
    ctor.argtypes = [C.c_void_p, C.c_void_p]
    ctor(C.addressof(ks), C.addressof(k))
    return ks


def test_round_key_schedule_constructor_is_host_key_expansion(aeslib, orc):
    fips = bytes.fromhex("2b7e151628aed2a6abf7158809cf4f3c")
    ks = bytes(_schedule(aeslib, fips))
    assert ks[16:20].hex() == "a0fafe17"  # w4 (test_aes.cpp:126-134)
    assert bytes(_schedule(aeslib, bytes(16)))[16:32].hex() == "62636363" * 4  # zero key, round 1
    assert ks == orc.expand_key(fips)


def test_sbox_tables(aeslib, orc):
    for name, inverse in ((SBOX, False), (INV_SBOX, True)):
        fn = getattr(aeslib, name)
        fn.restype = C.POINTER(C.c_uint8 * 256)
        t = bytes(fn().contents)
        assert t == (orc.inv_sbox() if inverse else orc.sbox())
    fn = getattr(aeslib, SBOX)
    assert bytes(fn().contents)[0x00] == 0x63 and bytes(fn().contents)[0x53] == 0xED


@pytest.mark.gpu
def test_bulk_and_block_entries_on_b200(aeslib, orc, gpu):
    key = bytes.fromhex("000102030405060708090a0b0c0d0e0f")
    ks = _schedule(aeslib, key)
    f = getattr(aeslib, ENC_ECB)
    g = getattr(aeslib, DEC_ECB)
    for fn in (f, g):
        fn.restype = None
        fn.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t, C.c_void_p]
    for n in (16, 4096, (3 << 20) + 48):
        data = os.urandom(n)
        src = C.create_string_buffer(data, n)
        dst = C.create_string_buffer(n)
        f(C.addressof(src), n, C.addressof(dst), n, C.addressof(ks))
        assert dst.raw == orc.ecb(0, data, key)
        back = C.create_string_buffer(n)
        g(C.addressof(dst), n, C.addressof(back), n, C.addressof(ks))
        assert back.raw == data
    # in-place (exact aliasing is legal, aes.hpp:84-85)
    data = os.urandom(1 << 20)
    buf = C.create_string_buffer(data, len(data))
    f(C.addressof(buf), len(data), C.addressof(buf), len(data), C.addressof(ks))
    assert buf.raw == orc.ecb(0, data, key)
    # FIPS-197 C.1 through encrypt_block (Block const& -> Block)
    blk = getattr(aeslib, ENC_BLOCK)
    blk.restype = State
    blk.argtypes = [C.c_void_p, C.c_void_p]
    pt = (C.c_uint8 * 16).from_buffer_copy(bytes.fromhex("00112233445566778899aabbccddeeff"))
    assert bytes(blk(C.addressof(pt), C.addressof(ks)).cells).hex() == "69c4e0d86a7b0430d8cdb78070b4c55a"
    # State by value in, State by value out (mix_columns KAT, test_aes.cpp:191-237)
    mix, inv = getattr(aeslib, MIX), getattr(aeslib, INV_MIX)
    for fn in (mix, inv):
        fn.restype = State
        fn.argtypes = [State]
    s = State()
    s.cells[:] = list(bytes.fromhex("db135345" * 4))
    out = mix(s)
    assert bytes(out.cells)[:4].hex() == "8e4da1bc"
    assert bytes(inv(out).cells) == bytes(s.cells)
