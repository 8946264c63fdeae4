"""TEST INFRASTRUCTURE ONLY -- ctypes loader for the CPU oracle.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this package.  The product package
(``paper_1403_7295_b200``) never does; see ``aes_oracle.c`` for what is
restated from where.

Two checkers live here:

* ``Oracle``  -- ``build/liboracle_aes.so``, the plain-C restatement of the
  reference's AES-128 / PKCS#7 / chunk-planner / sweep-generator path.
* ``RefLib``  -- ``_ref/libpaes_ref.so``, the reference's own ``paes_core``
  compiled from its sources by ``oracle/Makefile`` (present when the reference
  tree was available at build time; the .so travels to the GPU box).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "liboracle_aes.so")
REF_SO = os.path.join(HERE, "_ref", "libpaes_ref.so")

EINVAL = -22
EBADMSG = -74
EIO = -5
EWORKER = -1001


def build(quiet: bool = True) -> None:
    """Compile the oracle (and oracle/_ref when /root/reference exists)."""
    out = subprocess.run(["make", "-C", HERE], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


class ChunkSpec(C.Structure):
    _fields_ = [("offset", C.c_uint64), ("raw_len", C.c_uint64), ("padded_len", C.c_uint64),
                ("is_final", C.c_int32), ("_pad", C.c_int32)]


def _buf(data: bytes | bytearray | memoryview):
    if isinstance(data, (bytes, bytearray)):
        n = len(data)
        return (C.c_uint8 * max(n, 1)).from_buffer_copy(bytes(data) if n else b"\0"), n
    raise TypeError(type(data))


def _u8p(x):
    return C.cast(x, C.POINTER(C.c_uint8))


class Oracle:
    """The C restatement (oracle/aes_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        self.L = L
        u8p, u64 = C.POINTER(C.c_uint8), C.c_uint64
        L.oracle_expand_key.argtypes = [u8p, u8p]
        L.oracle_encrypt_block.argtypes = [u8p, u8p, u8p]
        L.oracle_decrypt_block.argtypes = [u8p, u8p, u8p]
        L.oracle_ecb.argtypes = [C.c_int, C.c_void_p, C.c_void_p, u64, u8p, C.c_int]
        L.oracle_ecb.restype = C.c_int
        L.oracle_encrypt_chunk.argtypes = [C.c_void_p, u64, C.c_int, u8p, C.c_void_p, C.POINTER(u64), C.c_int]
        L.oracle_decrypt_chunk.argtypes = [C.c_void_p, u64, C.c_int, u8p, C.c_void_p, C.POINTER(u64), C.c_int]
        L.oracle_unpad_final.argtypes = [C.c_void_p, u64]
        L.oracle_unpad_final.restype = C.c_int64
        L.oracle_plan_chunks.argtypes = [u64, C.c_uint32, C.POINTER(ChunkSpec), u64]
        L.oracle_plan_chunks.restype = C.c_int64
        L.oracle_plan_decrypt_chunks.argtypes = [u64, C.c_uint32, C.POINTER(ChunkSpec), u64]
        L.oracle_plan_decrypt_chunks.restype = C.c_int64
        L.oracle_sweep.argtypes = [u64, u64, C.c_void_p]
        L.oracle_batch_lengths.argtypes = [u64, C.c_uint32, C.POINTER(u64)]
        L.oracle_counter_fill.argtypes = [u64, u64, u64, C.c_void_p]
        L.oracle_checksum.argtypes = [C.c_void_p, u64, u64]
        L.oracle_checksum.restype = C.c_uint64
        L.oracle_round_transform.argtypes = [C.c_int, u8p, u8p]
        L.oracle_sbox.argtypes = [u8p]
        L.oracle_inv_sbox.argtypes = [u8p]
        L.oracle_gf_mul.argtypes = [C.c_uint8, C.c_uint8]
        L.oracle_gf_mul.restype = C.c_uint8

    # -- key schedule / blocks
    def expand_key(self, key: bytes) -> bytes:
        assert len(key) == 16
        k = (C.c_uint8 * 16).from_buffer_copy(key)
        rk = (C.c_uint8 * 176)()
        self.L.oracle_expand_key(k, rk)
        return bytes(rk)

    def _rk(self, key: bytes):
        return (C.c_uint8 * 176).from_buffer_copy(self.expand_key(key))

    def encrypt_block(self, block: bytes, key: bytes) -> bytes:
        i = (C.c_uint8 * 16).from_buffer_copy(block)
        o = (C.c_uint8 * 16)()
        self.L.oracle_encrypt_block(i, o, self._rk(key))
        return bytes(o)

    def decrypt_block(self, block: bytes, key: bytes) -> bytes:
        i = (C.c_uint8 * 16).from_buffer_copy(block)
        o = (C.c_uint8 * 16)()
        self.L.oracle_decrypt_block(i, o, self._rk(key))
        return bytes(o)

    def transform(self, which: int, state: bytes, rk16: bytes = bytes(16)) -> bytes:
        s = (C.c_uint8 * 16).from_buffer_copy(state)
        self.L.oracle_round_transform(which, s, (C.c_uint8 * 16).from_buffer_copy(rk16))
        return bytes(s)

    def sbox(self) -> bytes:
        o = (C.c_uint8 * 256)()
        self.L.oracle_sbox(o)
        return bytes(o)

    def inv_sbox(self) -> bytes:
        o = (C.c_uint8 * 256)()
        self.L.oracle_inv_sbox(o)
        return bytes(o)

    # -- bulk
    def ecb(self, direction: int, data, key: bytes, threads: int = 1) -> bytes:
        n = len(data)
        src = (C.c_uint8 * max(n, 1)).from_buffer_copy(bytes(data) if n else b"\0")
        dst = (C.c_uint8 * max(n, 1))()
        rc = self.L.oracle_ecb(direction, src, dst, n, self._rk(key), threads)
        if rc == EINVAL:
            raise ValueError("length must be a multiple of 16")
        return bytes(dst)[:n]

    def ecb_into(self, direction: int, src_ptr: int, dst_ptr: int, n: int, key: bytes, threads: int = 1) -> None:
        rc = self.L.oracle_ecb(direction, C.c_void_p(src_ptr), C.c_void_p(dst_ptr), n, self._rk(key), threads)
        if rc:
            raise ValueError("oracle_ecb rc=%d" % rc)

    def encrypt_chunk(self, data, is_final: bool, key: bytes, threads: int = 1) -> bytes:
        n = len(data)
        src = (C.c_uint8 * max(n, 1)).from_buffer_copy(bytes(data) if n else b"\0")
        dst = (C.c_uint8 * (n + 16))()
        ol = C.c_uint64()
        rc = self.L.oracle_encrypt_chunk(src, n, int(is_final), self._rk(key), dst, C.byref(ol), threads)
        if rc == EINVAL:
            raise ValueError("non-final chunk length must be a multiple of 16")
        return bytes(dst)[: ol.value]

    def decrypt_chunk(self, data, is_final: bool, key: bytes, threads: int = 1) -> bytes:
        n = len(data)
        src = (C.c_uint8 * max(n, 1)).from_buffer_copy(bytes(data) if n else b"\0")
        dst = (C.c_uint8 * max(n, 1))()
        ol = C.c_uint64()
        rc = self.L.oracle_decrypt_chunk(src, n, int(is_final), self._rk(key), dst, C.byref(ol), threads)
        if rc == EBADMSG:
            raise ValueError("padding error")
        if rc == EINVAL:
            raise ValueError("length must be a multiple of 16")
        return bytes(dst)[: ol.value]

    def unpad(self, data: bytes) -> int:
        n = len(data)
        src = (C.c_uint8 * max(n, 1)).from_buffer_copy(bytes(data) if n else b"\0")
        return int(self.L.oracle_unpad_final(src, n))

    # -- planner
    def plan(self, direction: int, total_len: int, workers: int):
        cap = max(1, min(workers, total_len // 16 + 1))
        arr = (ChunkSpec * cap)()
        fn = self.L.oracle_plan_chunks if direction == 0 else self.L.oracle_plan_decrypt_chunks
        n = fn(total_len, workers, arr, cap)
        if n < 0:
            return int(n)
        return [(c.offset, c.raw_len, c.padded_len, bool(c.is_final)) for c in arr[:n]]

    # -- inputs
    def sweep(self, seed: int, size: int) -> bytes:
        buf = (C.c_uint8 * max(size, 1))()
        self.L.oracle_sweep(seed, size, buf)
        return bytes(buf)[:size]

    def sweep_into(self, seed: int, size: int, ptr: int) -> None:
        self.L.oracle_sweep(seed, size, C.c_void_p(ptr))

    def counter_fill(self, seed: int, offset: int, size: int) -> bytes:
        buf = (C.c_uint8 * max(size, 1))()
        assert self.L.oracle_counter_fill(seed, offset, size, buf) == 0
        return bytes(buf)[:size]

    def checksum(self, data, base_word: int = 0) -> int:
        n = len(data)
        src = (C.c_uint8 * max(n, 1)).from_buffer_copy(bytes(data) if n else b"\0")
        return int(self.L.oracle_checksum(src, n, base_word))

    def checksum_ptr(self, ptr: int, n: int, base_word: int = 0) -> int:
        return int(self.L.oracle_checksum(C.c_void_p(ptr), n, base_word))

    def counter_fill_into(self, seed: int, offset: int, size: int, ptr: int) -> None:
        assert self.L.oracle_counter_fill(seed, offset, size, C.c_void_p(ptr)) == 0

    def batch_lengths(self, seed: int, n: int):
        arr = (C.c_uint64 * n)()
        self.L.oracle_batch_lengths(seed, n, arr)
        return list(arr)


class RefLib:
    """The reference's own paes_core, compiled from its sources (oracle/_ref)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = C.CDLL(path)
        self.L = L
        u8p, u64 = C.POINTER(C.c_uint8), C.c_uint64
        L.ref_expand_key.argtypes = [u8p, u8p]
        L.ref_encrypt_block.argtypes = [u8p, u8p, u8p]
        L.ref_decrypt_block.argtypes = [u8p, u8p, u8p]
        L.ref_ecb.argtypes = [C.c_int, C.c_void_p, C.c_void_p, u64, u8p]
        L.ref_chunk.argtypes = [C.c_int, C.c_void_p, u64, C.c_int, u8p, C.c_void_p, C.POINTER(u64)]
        L.ref_threads.argtypes = [C.c_int, C.c_void_p, u64, u8p, C.c_void_p, C.POINTER(u64), C.c_uint]
        L.ref_plan.argtypes = [C.c_int, u64, C.c_uint, C.POINTER(ChunkSpec), u64]
        L.ref_plan.restype = C.c_longlong
        L.ref_unpad.argtypes = [C.c_void_p, u64]
        L.ref_unpad.restype = C.c_longlong
        L.ref_sweep.argtypes = [u64, u64, C.c_void_p, C.c_char_p]
        L.ref_reject_outliers.argtypes = [C.POINTER(C.c_double), u64, C.POINTER(C.c_double), C.POINTER(u64)]
        L.ref_logical_cores.restype = C.c_uint
        L.ref_physical_cores.restype = C.c_uint
        L.ref_run_job.argtypes = [C.c_char_p, C.c_char_p, u8p, C.c_uint, C.c_int, C.c_int,
                                  C.POINTER(u64), C.POINTER(u64), C.POINTER(C.c_double)]
        L.ref_run_job_ex.argtypes = [C.c_char_p, C.c_char_p, u8p, C.c_uint, C.c_int, C.c_int, C.c_char_p,
                                     C.POINTER(u64), C.POINTER(u64), C.POINTER(C.c_double)]

    @staticmethod
    def _k(key: bytes):
        return (C.c_uint8 * 16).from_buffer_copy(key)

    def expand_key(self, key: bytes) -> bytes:
        rk = (C.c_uint8 * 176)()
        assert self.L.ref_expand_key(self._k(key), rk) == 0
        return bytes(rk)

    def encrypt_block(self, block: bytes, key: bytes) -> bytes:
        o = (C.c_uint8 * 16)()
        self.L.ref_encrypt_block((C.c_uint8 * 16).from_buffer_copy(block), o, self._k(key))
        return bytes(o)

    def decrypt_block(self, block: bytes, key: bytes) -> bytes:
        o = (C.c_uint8 * 16)()
        self.L.ref_decrypt_block((C.c_uint8 * 16).from_buffer_copy(block), o, self._k(key))
        return bytes(o)

    def ecb(self, direction: int, data: bytes, key: bytes) -> bytes:
        n = len(data)
        src = (C.c_uint8 * max(n, 1)).from_buffer_copy(bytes(data) if n else b"\0")
        dst = (C.c_uint8 * max(n, 1))()
        rc = self.L.ref_ecb(direction, src, dst, n, self._k(key))
        if rc:
            raise ValueError("ref_ecb rc=%d" % rc)
        return bytes(dst)[:n]

    def chunk(self, direction: int, data: bytes, is_final: bool, key: bytes):
        """Returns bytes, or a negative error code (EINVAL / EBADMSG)."""
        n = len(data)
        src = (C.c_uint8 * max(n, 1)).from_buffer_copy(bytes(data) if n else b"\0")
        dst = (C.c_uint8 * (n + 16))()
        ol = C.c_uint64()
        rc = self.L.ref_chunk(direction, src, n, int(is_final), self._k(key), dst, C.byref(ol))
        if rc:
            return rc
        return bytes(dst)[: ol.value]

    def threads_into(self, direction: int, src_ptr: int, n: int, key: bytes, dst_ptr: int, workers: int) -> int:
        ol = C.c_uint64()
        rc = self.L.ref_threads(direction, C.c_void_p(src_ptr), n, self._k(key), C.c_void_p(dst_ptr),
                                C.byref(ol), workers)
        if rc:
            raise RuntimeError("ref_threads rc=%d" % rc)
        return ol.value

    def plan(self, direction: int, total_len: int, workers: int):
        cap = max(1, min(workers, total_len // 16 + 1))
        arr = (ChunkSpec * cap)()
        n = self.L.ref_plan(direction, total_len, workers, arr, cap)
        if n < 0:
            return int(n)
        return [(c.offset, c.raw_len, c.padded_len, bool(c.is_final)) for c in arr[:n]]

    def unpad(self, data: bytes) -> int:
        n = len(data)
        src = (C.c_uint8 * max(n, 1)).from_buffer_copy(bytes(data) if n else b"\0")
        return int(self.L.ref_unpad(src, n))

    def sweep(self, seed: int, size: int) -> bytes:
        buf = (C.c_uint8 * max(size, 1))()
        fd, path = tempfile.mkstemp(prefix="paes_sweep_", dir="/dev/shm" if os.path.isdir("/dev/shm") else None)
        os.close(fd)
        try:
            assert self.L.ref_sweep(seed, size, buf, path.encode()) == 0
        finally:
            if os.path.exists(path):
                os.unlink(path)
        return bytes(buf)[:size]

    def reject_outliers(self, samples):
        n = len(samples)
        arr = (C.c_double * n)(*samples)
        out = (C.c_double * n)()
        m = C.c_uint64()
        rc = self.L.ref_reject_outliers(arr, n, out, C.byref(m))
        if rc:
            raise ValueError("no samples")
        return list(out[: m.value])

    def run_job(self, in_path: str, out_path: str, key: bytes, workers: int, strategy: int, direction: int,
                worker_exe: str = ""):
        """paes::run_job (strategy 0 sequential, 1 threads, 2 processes); returns
        (rc, bytes_in, bytes_out, seconds)."""
        bi, bo, sec = C.c_uint64(), C.c_uint64(), C.c_double()
        rc = self.L.ref_run_job_ex(in_path.encode(), out_path.encode(), self._k(key), workers, strategy, direction,
                                   worker_exe.encode(), C.byref(bi), C.byref(bo), C.byref(sec))
        return rc, bi.value, bo.value, sec.value

    def cores(self):
        return int(self.L.ref_physical_cores()), int(self.L.ref_logical_cores())


def ref_available() -> bool:
    return os.path.exists(REF_SO)
