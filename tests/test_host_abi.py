"""CPU-only: the C-ABI library loads and exports every declared symbol, and
its host-side rules (key expansion, planner/sharder, PKCS#7, seeded inputs,
checksums) match the oracle and the reference's golden vectors.  No kernel
is launched here."""
from __future__ import annotations

import ctypes as C
import os
import random
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "paes_cuda.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(paes_cuda_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol(lib):
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    from paper_1403_7295_b200 import _native

    assert sorted(n for n, _, _ in _native.SIGNATURES) == syms


def test_library_is_sm100a_and_not_a_fallback():
    from paper_1403_7295_b200 import _native

    path = _native.lib_path()
    blob = open(path, "rb").read()
    assert b"sm_100a" in blob  # embedded cubin for the right arch
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", path], capture_output=True, text=True)
    if out.returncode == 0:
        assert "sm_100a" in out.stdout


def test_no_oracle_in_product():
    """The product package never imports/links the oracle."""
    pkg = os.path.join(ROOT, "paper_1403_7295_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".hpp")):
                text = open(os.path.join(dirpath, f), errors="ignore").read()
                assert "import oracle" not in text and "liboracle" not in text and "libpaes_ref" not in text, f


def test_version(paes):
    assert "sm_100a" in paes.version()


def test_expand_key_matches_golden(paes, golden):
    for e in golden["key_schedules"]:
        assert paes.round_keys(bytes.fromhex(e["key"])).hex() == e["rk"]
    keys = paes.expand_key(bytes.fromhex("000102030405060708090a0b0c0d0e0f"))
    assert len(keys) == 11 and keys[0].hex() == "000102030405060708090a0b0c0d0e0f"  # test_smoke.py:21-25
    assert paes.expand_key(bytes(16))[1].hex() == "62636363" * 4
    with pytest.raises(ValueError):
        paes.round_keys(b"short")


def test_random_key_schedules_vs_oracle(paes, orc):
    rnd = random.Random(9)
    for _ in range(200):
        k = bytes(rnd.randrange(256) for _ in range(16))
        assert paes.round_keys(k) == orc.expand_key(k)


def test_plan_chunks_examples(paes, golden):
    """test_chunk.cpp:57-103 + golden grid from the reference's _paes.plan_chunks."""
    assert [c["raw_len"] for c in paes.plan_chunks(1000, 4)] == [256, 256, 256, 232]
    assert paes.plan_chunks(1000, 4)[-1]["padded_len"] == 240
    assert len(paes.plan_chunks(16, 33)) == 1 and len(paes.plan_chunks(17, 33)) == 2
    assert paes.plan_chunks(0, 33) == [{"offset": 0, "raw_len": 0, "padded_len": 16, "is_final": True}]
    assert len(paes.plan_chunks(1024, 65)) == 64  # chunk cap = data blocks (Appendix C.1)
    for e in golden["plans"]:
        got = [[c["offset"], c["raw_len"], c["padded_len"], c["is_final"]] for c in paes.plan_chunks(e["total"], e["workers"])]
        assert got == e["chunks"], (e["total"], e["workers"])
    with pytest.raises(ValueError):
        paes.plan_chunks(100, 0)


def test_plan_grid_vs_oracle(paes, orc):
    for total in range(0, 513, 5):
        for w in range(1, 18):
            got = [(c["offset"], c["raw_len"], c["padded_len"], c["is_final"]) for c in paes.plan_chunks(total, w)]
            assert got == orc.plan(0, total, w)
            if total and total % 16 == 0:
                got = [(c["offset"], c["raw_len"], c["padded_len"], c["is_final"])
                       for c in paes.plan_decrypt_chunks(total, w)]
                assert got == orc.plan(1, total, w)


def test_plan_decrypt_errors(paes):
    """test_chunk.cpp:165-176."""
    p = paes.plan_decrypt_chunks(1008, 4)
    assert [c["raw_len"] for c in p] == [256, 256, 256, 240] and p[-1]["is_final"]
    with pytest.raises(paes.PaddingError):
        paes.plan_decrypt_chunks(0, 2)
    with pytest.raises(paes.PaddingError):
        paes.plan_decrypt_chunks(100, 2)
    with pytest.raises(ValueError):
        paes.plan_decrypt_chunks(1008, 0)


def test_shards_cover_64gib_at_1_2_4_8(paes):
    """The multi-GPU sharder on the config-4 size: contiguous, 16-B aligned, pad on the last."""
    total = 64 << 30
    for n in (1, 2, 4, 8):
        p = paes.plan_chunks(total, n)
        assert len(p) == n
        off = 0
        for i, c in enumerate(p):
            assert c["offset"] == off and c["raw_len"] % 16 == 0
            off += c["raw_len"]
            assert c["is_final"] == (i == n - 1)
        assert off == total and p[-1]["padded_len"] == p[-1]["raw_len"] + 16


def test_pad_unpad(paes, golden):
    """test_chunk.cpp:128-163 + golden."""
    assert paes.pkcs7_pad(b"") == b"\x10" * 16
    assert paes.pkcs7_unpad(paes.pkcs7_pad(b"abc")) == b"abc"
    for e in golden["pad"]:
        assert paes.pkcs7_pad(bytes.fromhex(e["in"])).hex() == e["out"]
    for e in golden["unpad"]:
        data = bytes.fromhex(e["in"])
        if e["ok"]:
            assert paes.pkcs7_unpad(data).hex() == e["out"]
        else:
            with pytest.raises(ValueError):
                paes.pkcs7_unpad(data)
    for n in range(0, 65):
        data = bytes((i * 7 + 1) & 0xFF for i in range(n))
        assert paes.pkcs7_unpad(paes.pkcs7_pad(data)) == data


def test_reject_outliers_golden(paes, golden):
    for e in golden["reject_outliers"]:
        assert paes.reject_outliers(e["in"]) == pytest.approx(e["out"])
    with pytest.raises(ValueError):
        paes.reject_outliers([])


def test_sweep_generator_matches_oracle(paes, orc):
    assert paes.sweep(0, 16).hex() == "4c287f4282c15e6cfda0c041590ebc2a"
    for seed, n in [(0, 0), (1, 7), (2, 1031), (3, 16), ((4 << 32) + 9, 4096), (123, 100_001)]:
        assert paes.sweep(seed, n) == orc.sweep(seed, n)


def test_batch_lengths_and_counter_stream(paes, orc):
    lens = paes.batch_lengths(4, 4096)
    assert lens == orc.batch_lengths(4, 4096)
    assert all(4096 <= L <= 4 << 20 and L % 16 == 0 for L in lens)
    assert 1.8 * (1 << 30) < sum(lens) < 2.8 * (1 << 30)  # ~2.31 GiB expected
    for off, n in [(0, 64), (8, 40), (4096, 1000), ((64 << 30) - 64, 64)]:
        assert paes.counter_fill(3, off, n) == orc.counter_fill(3, off, n)
    data = paes.counter_fill(3, 0, 1 << 16)
    assert paes.checksum(data, 0) == orc.checksum(data, 0)
    # additivity: shard checksums sum to the whole
    a, b = data[: 1 << 15], data[1 << 15:]
    assert (paes.checksum(a, 0) + paes.checksum(b, (1 << 15) // 8)) % (1 << 64) == paes.checksum(data, 0)


def test_compute_without_gpu_fails_loudly(paes):
    if paes.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(paes.GpuError):
        paes.encrypt_bytes(b"abc", bytes(16))
    with pytest.raises(paes.GpuError):
        paes.ecb_device(0, 0x1000, 0x1000, 16, paes.round_keys(bytes(16)))


def test_argument_errors_before_device(paes):
    with pytest.raises(ValueError):
        paes.encrypt_ecb(bytes(15), bytes(16))
    with pytest.raises(ValueError):
        paes.encrypt_chunk(bytes(17), False, bytes(16))
    with pytest.raises(paes.PaddingError):
        paes.decrypt_bytes(b"", bytes(16))
    with pytest.raises(ValueError, match="strategy must be"):
        paes.encrypt_file("/nonexistent", "/tmp/x", bytes(16), strategy="fibers")
    # the reference's worker-count rule for its parallel strategies (exec.cpp:209, 273)
    with pytest.raises(ValueError, match="run_threaded: workers must be >= 1"):
        paes.encrypt_file("/nonexistent", "/tmp/x", bytes(16), workers=0, strategy="threads")
    with pytest.raises(ValueError, match="run_process_isolated: workers must be >= 1"):
        paes.decrypt_file("/nonexistent", "/tmp/x", bytes(16), workers=0, strategy="processes")
    from paper_1403_7295_b200 import _native as N

    L = N.load()
    assert L.paes_cuda_ecb(7, None, None, 0, paes.round_keys(bytes(16)), 0) == N.EINVAL
    assert L.paes_cuda_set_pipeline(15, 0) == N.EINVAL
    assert b"multiple of 16" in L.paes_cuda_last_error()
    assert L.paes_cuda_set_pipeline(16, 0) == N.EINVAL  # below the 4 KiB floor
    assert L.paes_cuda_set_pipeline(0, 33) == N.EINVAL
    assert L.paes_cuda_set_pipeline(0, -1) == N.EINVAL
    assert L.paes_cuda_set_pipeline(0, 0) == 0  # 0 keeps the current values


def test_paes_alias_module(paes):
    """`import _paes` from the compat directory is this engine under the reference's module name."""
    import importlib
    import sys

    compat = os.path.join(os.path.dirname(paes.__file__), "compat")
    sys.path.insert(0, compat)
    try:
        sys.modules.pop("_paes", None)
        alias = importlib.import_module("_paes")
    finally:
        sys.path.remove(compat)
        sys.modules.pop("_paes", None)
    for name in ("encrypt_block", "decrypt_block", "expand_key", "encrypt_bytes", "decrypt_bytes", "pkcs7_pad",
                 "pkcs7_unpad", "plan_chunks", "reject_outliers", "encrypt_file", "decrypt_file", "csv_header",
                 "PaddingError", "WorkerError", "IoError"):
        assert getattr(alias, name) is getattr(paes, name), name
    assert alias.expand_key(bytes(16))[1].hex() == "62636363" * 4  # test_aes.cpp:120-124
    assert [c["raw_len"] for c in alias.plan_chunks(1000, 4)] == [256, 256, 256, 232]  # test_smoke.py:48-53


def test_missing_library_raises(tmp_path, monkeypatch):
    from paper_1403_7295_b200 import _native

    monkeypatch.setattr(_native, "_lib", None)
    monkeypatch.setattr(_native, "lib_path", lambda: str(tmp_path / "nope.so"))
    with pytest.raises(_native.NativeLibraryMissing):
        _native.load()


def test_batch_descriptor_errors_before_device(paes):
    """plan_batch validates every descriptor before touching a device."""
    rk = paes.round_keys(bytes(16))
    with pytest.raises(ValueError, match="overflows"):
        paes.ecb_batch(0, 1, 1, [(1 << 64) - 16], [0], [32], rk, True)
    with pytest.raises(ValueError, match="overflows"):
        paes.ecb_batch_host(0, 1, 1, [0], [(1 << 64) - 16], [16], rk, True)
    with pytest.raises(paes.PaddingError):
        paes.ecb_batch(1, 1, 1, [0], [0], [0], rk, True)
    assert paes.ecb_batch(0, 0, 0, [], [], [], b"", True) == []


def test_sbox_tables_match_oracle(paes, orc):
    """sbox()/inv_sbox() (aes.hpp:69-70) are the library's compile-time tables."""
    assert paes.sbox() == orc.sbox()
    assert paes.sbox(inverse=True) == orc.inv_sbox()
    assert paes.sbox()[0x00] == 0x63 and paes.sbox()[0x53] == 0xED


def test_state_transform_errors_before_device(paes):
    with pytest.raises(ValueError):
        paes.state_transform(paes.SUB_BYTES, bytes(15))
    with pytest.raises(ValueError):
        paes.state_transform(9, bytes(16))
    with pytest.raises(ValueError):
        paes.state_transform(paes.ADD_ROUND_KEY, bytes(16))  # no round key
    assert paes.state_transform(paes.MIX_COLUMNS, b"") == b""


def test_python_wrappers_check_what_the_abi_cannot(paes):
    """Bare pointers cross the ABI, so the Python layer checks sizes first."""
    rk = paes.round_keys(bytes(16))
    with pytest.raises(ValueError, match="176 bytes per message"):
        paes.ecb_batch(0, 1, 1, [0, 16], [0, 32], [16, 16], rk, True)  # one schedule for two messages
    with pytest.raises(ValueError, match="same length"):
        paes.ecb_batch_host(0, 1, 1, [0], [0, 16], [16], rk, True)
    with pytest.raises(ValueError, match="176 bytes per message"):
        paes.BatchPlan(0, [0], [0], [16], rk[:100], True)
    with pytest.raises(ValueError, match="176-byte"):
        paes.ecb_device(0, 1, 1, 16, bytes(16))
    with pytest.raises(ValueError, match="176-byte"):
        paes.chunk_device(0, 1, 16, True, rk + b"x", 1)


def test_partial_overlap_is_rejected_before_any_device_work(lib):
    """in/out may alias exactly (aes.hpp:84-85) or be disjoint; a partial
    overlap is PAES_EINVAL, decided on the host (this runs without a GPU)."""
    from paper_1403_7295_b200 import _native as N

    rk = (C.c_uint8 * 176)()
    buf = (C.c_uint8 * 4096)()
    base = C.addressof(buf)
    olen = C.c_uint64()
    res = (C.c_uint64 * 1)()
    # device-pointer entries: the check precedes the device lookup
    assert lib.paes_cuda_ecb_device(0, base, base + 16, 256, rk, 0, None) == N.EINVAL
    assert "alias" in N.last_error()
    assert lib.paes_cuda_ecb_device(1, base + 32, base, 256, rk, 0, None) == N.EINVAL
    assert lib.paes_cuda_chunk_device(0, base, 100, 1, rk, base + 48, C.byref(olen), 0, None) == N.EINVAL
    # out is the padded length (112 B here), so an input starting at out + 104 overlaps it
    assert lib.paes_cuda_chunk_device(0, base + 104, 100, 1, rk, base, C.byref(olen), 0, None) == N.EINVAL
    assert lib.paes_cuda_chunk_device_async(1, base, 256, 1, rk, base + 128, res, 0, None) == N.EINVAL
    # host-pointer entries
    assert lib.paes_cuda_ecb(0, buf, C.cast(base + 16, C.POINTER(C.c_uint8)), 256, rk, 0) == N.EINVAL
    assert lib.paes_cuda_chunk(0, buf, 100, 1, rk, C.cast(base + 64, C.POINTER(C.c_uint8)), C.byref(olen), 0) == \
        N.EINVAL
    # the async entry needs an aligned result word
    assert lib.paes_cuda_chunk_device_async(0, base, 256, 1, rk, base + 1024, None, 0, None) == N.EINVAL
    assert lib.paes_cuda_chunk_device_async(0, base, 256, 1, rk, base + 1024, base + 2052, 0, None) == N.EINVAL
    # a zero-length final decrypt is unpad_final's PaddingError, before any data is read
    assert lib.paes_cuda_chunk_device_async(1, base, 0, 1, rk, base + 1024, res, 0, None) == N.EBADMSG


def test_product_library_links_no_reference_code():
    """libpaes_cuda.so is built from this repo's sources only: none of the
    reference's own symbols (paes::aes::*, paes::encrypt_chunk, ...) are in it,
    and it does not depend on the reference build in oracle/_ref."""
    import subprocess

    from paper_1403_7295_b200 import _native

    path = _native.lib_path()
    syms = subprocess.run(["nm", "-C", path], capture_output=True, text=True).stdout
    for bad in ("paes::aes::", "paes::encrypt_chunk", "paes::run_job", "paes::plan_chunks", "RoundKeySchedule"):
        assert bad not in syms, bad
    deps = subprocess.run(["ldd", path], capture_output=True, text=True).stdout
    assert "paes_ref" not in deps and "_paes" not in deps


def test_stale_library_warns_instead_of_loading_silently(monkeypatch):
    """load() says when libpaes_cuda.so is older than its sources (it never
    rebuilds behind the caller's back)."""
    import warnings

    from paper_1403_7295_b200 import _native
    from paper_1403_7295_b200 import build as B

    monkeypatch.setattr(_native, "_lib", None)
    monkeypatch.delenv("PAES_CUDA_LIB", raising=False)
    monkeypatch.setattr(B, "_stale", lambda: True)
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        L = _native.load()
    assert L is not None
    assert any("older than its sources" in str(x.message) for x in w)


def test_input_buffers_are_borrowed_whatever_their_kind(paes, tmp_path):
    """paes._InBuf: bytes, writable buffers and READ-ONLY buffers (memoryview
    of bytes, read-only numpy array, read-only mmap of a file) all reach the
    library by pointer -- a read-only buffer is not copied into a new bytes
    object first (that single-threaded copy would dominate a multi-GiB call)."""
    import mmap

    import numpy as np

    data = bytes(range(256)) * 5 + b"xyz"
    want = data + bytes([16 - len(data) % 16]) * (16 - len(data) % 16)
    ro = np.frombuffer(data, dtype=np.uint8)
    assert not ro.flags.writeable
    f = tmp_path / "in.bin"
    f.write_bytes(data)
    with open(f, "rb") as fh, mmap.mmap(fh.fileno(), 0, access=mmap.ACCESS_READ) as mm:
        for buf in (data, bytearray(data), memoryview(data), ro, mm, memoryview(bytearray(data))[:]):
            assert paes.pkcs7_pad(buf) == want, type(buf)
            b = paes._InBuf(buf)
            assert b.n == len(data)
            if not isinstance(buf, bytes):
                assert not isinstance(b.keep, bytes), type(buf)  # borrowed, not copied
            del b
    assert paes.pkcs7_pad(memoryview(b"")) == bytes([16]) * 16
