"""Python face of the engine, mirroring the reference's ``_paes`` module.

Same names, argument meaning and error behaviour as
proj/python/paes_module.cpp (see the per-function citations), so the
reference's own smoke tests read the same against this engine; every compute
call goes through the C ABI (include/paes_cuda.h) into the sm_100a kernels.
Every compute path is the GPU engine: ``strategy="gpu"`` names it, and the
reference's own "sequential"/"threads"/"processes" names are accepted too and
run the same GPU pipeline (their outputs are identical by the reference's own
tests), so callers need not change their arguments.

Exceptions (paes_module.cpp:153-155): PaddingError -> ValueError,
WorkerError -> RuntimeError, IoError -> OSError.  CUDA failures raise
GpuError (RuntimeError); invalid arguments raise ValueError as pybind11 maps
std::invalid_argument.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from typing import Iterable, List

from . import _native as N
from ._native import DECRYPT, ENCRYPT

BLOCK = 16


class PaddingError(ValueError):
    """Malformed PKCS#7 trailer (errors.hpp:24-27)."""


class WorkerError(RuntimeError):
    """One or more GPU shards failed; message names the chunk (errors.hpp:30-33)."""


class IoError(OSError):
    """File I/O failure (errors.hpp:13-21)."""


class GpuError(RuntimeError):
    """CUDA runtime failure or no usable device."""


def _raise(rc: int) -> None:
    if rc >= 0:
        return
    msg = N.last_error()
    if rc == N.EBADMSG:
        raise PaddingError(msg)
    if rc == N.EINVAL:
        raise ValueError(msg)
    if rc == N.EWORKER:
        raise WorkerError(msg)
    if rc == N.EIO:
        raise IoError(msg)
    raise GpuError(f"{msg} (code {rc})")


def _as_key(key: bytes) -> bytes:
    key = bytes(key)
    if len(key) != 16:
        raise ValueError("key must be exactly 16 bytes")
    return key


class _InBuf:
    """Borrow a read-only pointer to bytes-like data without copying."""

    def __init__(self, data):
        if isinstance(data, bytes):
            self.keep = data
            self.ptr = C.cast(C.c_char_p(data), C.c_void_p).value if data else None
            self.n = len(data)
            return
        mv = memoryview(data).cast("B")
        self.n = mv.nbytes
        if self.n == 0:
            self.keep, self.ptr = mv, None
        elif mv.readonly:
            # ctypes cannot borrow a read-only buffer (a read-only mmap, a
            # memoryview of bytes); numpy can, without the single-threaded
            # bytes(mv) copy that would dominate a multi-GiB call
            try:
                import numpy as np

                arr = np.frombuffer(mv, dtype=np.uint8)
                self.keep = (mv, arr)
                self.ptr = int(arr.ctypes.data)
            except ImportError:
                self.keep = bytes(mv)
                self.ptr = C.cast(C.c_char_p(self.keep), C.c_void_p).value
        else:
            arr = (C.c_uint8 * self.n).from_buffer(mv)
            self.keep = (mv, arr)
            self.ptr = C.addressof(arr)


_new_bytes_api = C.pythonapi.PyBytes_FromStringAndSize
_new_bytes_api.restype = C.py_object
_new_bytes_api.argtypes = [C.c_void_p, C.c_ssize_t]


class _OutBytes:
    """A fresh, not-yet-shared bytes object the library writes into directly,
    so a result reaches Python with no extra copy (the reference returns
    py::bytes too).  Sizes below 16 fall back to a ctypes buffer: CPython
    shares its empty bytes object."""

    def __init__(self, n: int):
        self.n = n
        if n >= BLOCK:
            self.obj = _new_bytes_api(None, n)  # uninitialised, refcount 1, hash not yet cached
            self.ptr = C.cast(C.c_char_p(self.obj), C.c_void_p).value
        else:
            self.obj = C.create_string_buffer(max(n, 1))
            self.ptr = C.addressof(self.obj)

    def result(self, m: int) -> bytes:
        if not isinstance(self.obj, bytes):
            return C.string_at(self.ptr, m)
        # an unpadded decrypt is 1-16 bytes short of the buffer: one slice copy
        return self.obj if m == self.n else self.obj[:m]


def round_keys(key: bytes) -> bytes:
    """176-byte expanded schedule (RoundKeySchedule, aes.cpp:151-180)."""
    key = _as_key(key)
    rk = (C.c_uint8 * 176)()
    _raise(N.load().paes_cuda_expand_key(key, rk))
    return bytes(rk)


def expand_key(key: bytes) -> List[bytes]:
    """11 round keys (paes_module.cpp:59-68)."""
    rk = round_keys(key)
    return [rk[16 * r:16 * r + 16] for r in range(11)]


# ---------------------------------------------------------------- single-state API
SUB_BYTES, INV_SUB_BYTES, SHIFT_ROWS, INV_SHIFT_ROWS, MIX_COLUMNS, INV_MIX_COLUMNS, ADD_ROUND_KEY = range(7)


def state_transform(op: int, states: bytes, rk16: bytes = None) -> bytes:
    """The reference's per-transform wrappers (aes.hpp:72-78, aes.cpp:194-227)
    applied on the GPU to len(states) // 16 independent states."""
    states = bytes(states)
    if len(states) % 16:
        raise ValueError("states must be a whole number of 16-byte states")
    if rk16 is not None and len(rk16) != 16:
        raise ValueError("round key must be 16 bytes")
    buf = (C.c_uint8 * max(len(states), 1)).from_buffer_copy(states or b"\0")
    _raise(N.load().paes_cuda_state_transform(op, buf, len(states) // 16, rk16))
    return bytes(buf)[: len(states)]


def sbox(inverse: bool = False) -> bytes:
    """sbox() / inv_sbox() (aes.hpp:69-70): the library's compile-time tables."""
    out = (C.c_uint8 * 256)()
    _raise(N.load().paes_cuda_sbox(int(bool(inverse)), out))
    return bytes(out)


# ---------------------------------------------------------------- bulk ECB
def ecb(direction: int, data, key: bytes, ngpus: int = 0) -> bytes:
    """aes::encrypt_ecb / decrypt_ecb (aes.hpp:86-89) over host memory."""
    rk = round_keys(key)
    src = _InBuf(data)
    out = _OutBytes(src.n)
    _raise(N.load().paes_cuda_ecb(direction, src.ptr, out.ptr, src.n, rk, ngpus))
    return out.result(src.n)


def encrypt_ecb(data, key: bytes, ngpus: int = 0) -> bytes:
    return ecb(ENCRYPT, data, key, ngpus)


def decrypt_ecb(data, key: bytes, ngpus: int = 0) -> bytes:
    return ecb(DECRYPT, data, key, ngpus)


def encrypt_block(block: bytes, key: bytes) -> bytes:
    """paes_module.cpp:70-75 (one block through the GPU path)."""
    if len(block) != 16:
        raise ValueError("block must be exactly 16 bytes")
    return ecb(ENCRYPT, bytes(block), key, 1)


def decrypt_block(block: bytes, key: bytes) -> bytes:
    if len(block) != 16:
        raise ValueError("block must be exactly 16 bytes")
    return ecb(DECRYPT, bytes(block), key, 1)


# ---------------------------------------------------------------- chunks
_TRIM_COPY_MAX = 256 * 1024  # a host copy of this many bytes costs about one short GPU call


def chunk(direction: int, data, is_final: bool, key: bytes, ngpus: int = 0) -> bytes:
    """encrypt_chunk / decrypt_chunk (exec.hpp:61-65) over host memory."""
    rk = round_keys(key)
    src = _InBuf(data)
    L = N.load()
    if direction == DECRYPT and is_final and src.n > _TRIM_COPY_MAX and src.n % BLOCK == 0:
        # Size the result exactly, so it needs no trimming copy: decrypt the
        # trailer block first (GPU), apply unpad_final's rule to it, then
        # decrypt the leading n-16 bytes as a non-final chunk straight into
        # the result and append the trailer's unpadded part.  (Up to
        # _TRIM_COPY_MAX bytes one call and a trimming copy are cheaper than
        # the extra call: decrypt_bytes of 16 KiB 42 -> ~27 us.)
        last = C.create_string_buffer(BLOCK)
        _raise(L.paes_cuda_ecb(DECRYPT, src.ptr + src.n - BLOCK, last, BLOCK, rk, 1))
        keep = L.paes_cuda_unpad_final(last, BLOCK)
        _raise(keep)  # PaddingError on a malformed trailer, as the in-kernel check would raise
        head = src.n - BLOCK
        out = _OutBytes(head + keep)
        olen = C.c_uint64()
        _raise(L.paes_cuda_chunk(DECRYPT, src.ptr, head, 0, rk, out.ptr, C.byref(olen), ngpus))
        C.memmove(out.ptr + head, last, keep)
        return out.result(head + keep)
    cap = (src.n // BLOCK + 1) * BLOCK if (direction == ENCRYPT and is_final) else src.n
    out = _OutBytes(cap)
    olen = C.c_uint64()
    _raise(L.paes_cuda_chunk(direction, src.ptr, src.n, int(bool(is_final)), rk, out.ptr, C.byref(olen), ngpus))
    return out.result(olen.value)


def encrypt_chunk(data, is_final: bool, key: bytes, ngpus: int = 0) -> bytes:
    return chunk(ENCRYPT, data, is_final, key, ngpus)


def decrypt_chunk(data, is_final: bool, key: bytes, ngpus: int = 0) -> bytes:
    return chunk(DECRYPT, data, is_final, key, ngpus)


def encrypt_bytes(data, key: bytes) -> bytes:
    """ECB over the PKCS#7-padded input (paes_module.cpp:84-88)."""
    return chunk(ENCRYPT, data, True, key)


def decrypt_bytes(data, key: bytes) -> bytes:
    """paes_module.cpp:90-93: raises PaddingError (ValueError) on a bad trailer."""
    return chunk(DECRYPT, data, True, key)


# ---------------------------------------------------------------- host rules
def pkcs7_pad(data) -> bytes:
    """pad_final (chunk.cpp:83-88)."""
    src = _InBuf(data)
    out = C.create_string_buffer(src.n + BLOCK)
    n = N.load().paes_cuda_pad_final(src.ptr, src.n, out)
    _raise(n)
    return out.raw[:n]


def pkcs7_unpad(data) -> bytes:
    """unpad_final (chunk.cpp:90-100)."""
    src = _InBuf(data)
    n = N.load().paes_cuda_unpad_final(src.ptr, src.n)
    _raise(n)
    return bytes(memoryview(data).cast("B")[:n]) if not isinstance(data, bytes) else data[:n]


def _plan(fn, total_len: int, workers: int):
    L = N.load()
    cap = max(1, min(int(workers), int(total_len) // 16 + 1))
    arr = (N.ChunkSpec * cap)()
    n = getattr(L, fn)(total_len, workers, arr, cap)
    _raise(n)
    return [{"offset": c.offset, "raw_len": c.raw_len, "padded_len": c.padded_len, "is_final": bool(c.is_final)}
            for c in arr[:n]]


def plan_chunks(total_len: int, workers: int):
    """plan_chunks (chunk.cpp:27-55) -- also the multi-GPU shard rule."""
    if workers < 0:
        raise ValueError("workers must be >= 1")
    return _plan("paes_cuda_plan_chunks", total_len, workers)


def plan_decrypt_chunks(cipher_len: int, workers: int):
    """plan_decrypt_chunks (chunk.cpp:57-81)."""
    if workers < 0:
        raise ValueError("workers must be >= 1")
    return _plan("paes_cuda_plan_decrypt_chunks", cipher_len, workers)


def reject_outliers(samples: Iterable[float]) -> List[float]:
    """Median/MAD filter of the bench harness (bench.cpp:49-79), restated."""
    s = [float(x) for x in samples]
    if not s:
        raise ValueError("reject_outliers: no samples")
    n = len(s)

    def median(v):
        v = sorted(v)
        return v[n // 2] if n % 2 else 0.5 * (v[n // 2 - 1] + v[n // 2])

    m = median(s)
    devs = [abs(x - m) for x in s]
    mad = median(devs)
    thr = 3.0 * mad if mad > 0.0 else 0.01 * abs(m)
    keep = [i for i in range(n) if devs[i] <= thr]
    floor = (n + 1) // 2
    if len(keep) < floor:
        order = sorted(range(n), key=lambda i: devs[i])  # stable: ties keep index order
        keep = sorted(order[:floor])
    return [s[i] for i in keep]


# ---------------------------------------------------------------- files
# The reference's CPU strategy names (strategy_from_string exec.cpp:33-38).
# They all produce the same bytes (test_smoke.py:77-78; test_exec.cpp:64-86),
# so a caller written against `_paes` keeps its strategy argument and runs on
# the GPU pipeline: `workers` there counts CPU workers, so it is clamped to
# the visible GPUs.  worker_exe only named the process strategy's worker
# binary and is not needed.
REFERENCE_STRATEGIES = ("sequential", "threads", "processes")


def _job(direction: int, input: str, output: str, key: bytes, workers: int, strategy: str, worker_exe: str):
    if strategy not in REFERENCE_STRATEGIES and strategy != "gpu":
        # to_strategy paes_module.cpp:43-46
        raise ValueError("strategy must be sequential, threads, processes or gpu")
    if workers < 0:
        raise ValueError("workers must be >= 0")
    if strategy in ("threads", "processes") and workers == 0:
        # run_threaded exec.cpp:209 / run_process_isolated exec.cpp:273
        raise ValueError(f"run_{'threaded' if strategy == 'threads' else 'process_isolated'}: workers must be >= 1")
    key = _as_key(key)
    if strategy == "sequential":
        workers = 1  # run_sequential exec.cpp:206 ignores workers
    elif strategy in REFERENCE_STRATEGIES:
        workers = max(1, min(workers, device_count()))
    o = N.JobOutcome()
    try:
        _raise(N.load().paes_cuda_run_job(os.fsencode(input), os.fsencode(output), key, workers, direction,
                                          C.byref(o)))
    except WorkerError as e:
        # run_sequential runs its one chunk inline, so a bad trailer surfaces
        # as the PaddingError itself, not wrapped (exec.cpp:184-186 vs :206)
        inner = str(e).split(": ", 2)[-1]
        if strategy == "sequential" and inner.startswith("unpad:"):
            raise PaddingError(inner) from None
        raise
    return {"bytes_in": o.bytes_in, "bytes_out": o.bytes_out, "seconds": o.seconds}


def encrypt_file(input: str, output: str, key: bytes, workers: int = 1, strategy: str = "sequential",
                 worker_exe: str = ""):
    """run_job(Encrypt) (paes_module.cpp:121-134), same defaults as the
    reference: strategy "sequential" (one GPU, a bad trailer raises the bare
    PaddingError); "gpu" takes workers = GPUs (0 = all)."""
    return _job(ENCRYPT, input, output, key, workers, strategy, worker_exe)


def decrypt_file(input: str, output: str, key: bytes, workers: int = 1, strategy: str = "sequential",
                 worker_exe: str = ""):
    """run_job(Decrypt) (paes_module.cpp:136-149); defaults as encrypt_file."""
    return _job(DECRYPT, input, output, key, workers, strategy, worker_exe)


# ---------------------------------------------------------------- device side
def device_count() -> int:
    return int(N.load().paes_cuda_device_count())


def set_devices(ids) -> None:
    ids = list(ids)
    arr = (C.c_int * max(len(ids), 1))(*ids)
    _raise(N.load().paes_cuda_set_devices(arr, len(ids)))


def set_pipeline(chunk_bytes: int = 0, streams: int = 0) -> None:
    _raise(N.load().paes_cuda_set_pipeline(chunk_bytes, streams))


def csv_header() -> str:
    """The bench report's CSV header (paes_module.cpp:151, report.hpp:12-13)."""
    from .report import CSV_HEADER

    return CSV_HEADER


DEFAULT_ZERO_COPY_MAX = 48 << 20  # the library's default (include/paes_cuda.h)


def set_zero_copy_max(nbytes: int) -> None:
    """Pinned host ranges up to ``nbytes`` run as one zero-copy kernel on the
    caller's buffers (0 = always use the copy-engine ring)."""
    _raise(N.load().paes_cuda_set_zero_copy_max(nbytes))


def _tensor_call(direction: int, x, key: bytes, is_final: bool, out):
    import torch

    if not (isinstance(x, torch.Tensor) and x.is_cuda and x.dtype == torch.uint8):
        raise ValueError("expected a CUDA uint8 tensor")
    x = x.contiguous().view(-1)
    n = x.numel()
    cap = (n // 16 + 1) * 16 if (direction == ENCRYPT and is_final) else n
    if out is None:
        out = torch.empty(max(cap, 1), dtype=torch.uint8, device=x.device)
    elif not (out.is_cuda and out.dtype == torch.uint8 and out.is_contiguous() and out.numel() >= cap):
        raise ValueError(f"out must be a contiguous CUDA uint8 tensor of >= {cap} elements")
    dev = x.device.index if x.device.index is not None else torch.cuda.current_device()
    stream = torch.cuda.current_stream(dev).cuda_stream
    m = chunk_device(direction, x.data_ptr(), n, is_final, round_keys(key), out.data_ptr(), dev, stream)
    return out[:m]


def encrypt_tensor(x, key: bytes, is_final: bool = True, out=None):
    """encrypt_chunk on a CUDA uint8 tensor, on the current torch stream;
    returns the ciphertext view (always-pad when is_final)."""
    return _tensor_call(ENCRYPT, x, key, is_final, out)


def decrypt_tensor(x, key: bytes, is_final: bool = True, out=None):
    """decrypt_chunk on a CUDA uint8 tensor; a final chunk's trailer is checked
    (PaddingError) and the returned view excludes the padding."""
    return _tensor_call(DECRYPT, x, key, is_final, out)


def ecb_device(direction: int, d_in: int, d_out: int, nbytes: int, rk: bytes, device: int = 0, stream: int = 0):
    """Device-resident ECB on raw pointers (asynchronous on `stream`)."""
    _raise(N.load().paes_cuda_ecb_device(direction, d_in, d_out, nbytes, _rk176(rk), device, stream or None))


_tls = threading.local()


def chunk_device(direction: int, d_in: int, nbytes: int, is_final: bool, rk: bytes, d_out: int, device: int = 0,
                 stream: int = 0) -> int:
    """encrypt_chunk / decrypt_chunk on device pointers (asynchronous on
    `stream` except a final decrypt, which returns the unpadded length)."""
    olen = getattr(_tls, "olen", None)
    if olen is None:
        olen = _tls.olen = C.c_uint64()
    rc = N.load().paes_cuda_chunk_device(direction, d_in, nbytes, 1 if is_final else 0, _rk176(rk), d_out,
                                         C.byref(olen), device, stream or None)
    if rc:
        _raise(rc)
    return olen.value


BAD_PAD = (1 << 64) - 1  # PAES_BAD_PAD: the result word of a final decrypt with a malformed trailer


def chunk_device_async(direction: int, d_in: int, nbytes: int, is_final: bool, rk: bytes, d_out: int, d_result: int,
                       device: int = 0, stream: int = 0) -> None:
    """Queued chunk transform (paes_cuda_chunk_device_async): never syncs, so
    it can be captured in a CUDA graph.  When it has run, the uint64 at
    ``d_result`` (device or mapped pinned memory) holds the output length --
    the unpadded length for a final decrypt -- or ``BAD_PAD``."""
    _raise(N.load().paes_cuda_chunk_device_async(direction, d_in, nbytes, int(bool(is_final)), _rk176(rk), d_out,
                                                 d_result, device, stream or None))


def _u64_array(xs):
    import numpy as np

    a = np.ascontiguousarray(np.asarray(xs, dtype=np.uint64))
    return a, a.ctypes.data_as(C.POINTER(C.c_uint64))


def _rk176(rk) -> bytes:
    """An expanded schedule crosses the ABI as a bare pointer: check its size here."""
    if type(rk) is bytes and len(rk) == 176:
        return rk
    rk = bytes(rk)
    if len(rk) != 176:
        raise ValueError("round keys must be the 176-byte expanded schedule (round_keys(key))")
    return rk


def _batch_arrays(in_off, out_off, lens, rks):
    """Descriptor arrays and per-message schedules for the batch calls; the C
    ABI takes bare pointers, so the counts are checked here."""
    n = len(lens)
    if len(in_off) != n or len(out_off) != n:
        raise ValueError("in_off, out_off and lens must have the same length")
    rks = bytes(rks)
    if len(rks) != 176 * n:
        raise ValueError(f"rks must hold 176 bytes per message ({176 * n}), got {len(rks)}")
    return n, [_u64_array(in_off), _u64_array(out_off), _u64_array(lens)], rks


def ecb_batch(direction: int, d_in: int, d_out: int, in_off, out_off, lens, rks: bytes, pad: bool, device: int = 0,
              stream: int = 0):
    """One fused launch over n messages with per-message keys (config 5)."""
    import numpy as np

    n, keep, rks = _batch_arrays(in_off, out_off, lens, rks)
    olens = np.zeros(max(n, 1), dtype=np.uint64)
    _raise(N.load().paes_cuda_ecb_batch(direction, d_in, d_out, keep[0][1], keep[1][1], keep[2][1], rks, n,
                                        int(bool(pad)), olens.ctypes.data_as(C.POINTER(C.c_uint64)), device,
                                        stream or None))
    return olens[:n].tolist()


def ecb_batch_host(direction: int, h_in: int, h_out: int, in_off, out_off, lens, rks: bytes, pad: bool,
                   device: int = 0):
    """Host-pointer batch (paes_cuda_batch_host): grouped, pipelined H2D /
    fused launch / D2H.  h_in / h_out are host addresses (pinned for speed)."""
    import numpy as np

    n, keep, rks = _batch_arrays(in_off, out_off, lens, rks)
    olens = np.zeros(max(n, 1), dtype=np.uint64)
    _raise(N.load().paes_cuda_batch_host(direction, h_in, h_out, keep[0][1], keep[1][1], keep[2][1], rks, n,
                                         int(bool(pad)), olens.ctypes.data_as(C.POINTER(C.c_uint64)), device))
    return olens[:n].tolist()


class BatchPlan:
    """Prepared batch (paes_cuda_batch_plan_*): descriptors and key words live
    on the device; run() is a single launch."""

    def __init__(self, direction: int, in_off, out_off, lens, rks: bytes, pad: bool, device: int = 0):
        self._h = None
        self.n, (a, b, c), rks = _batch_arrays(in_off, out_off, lens, rks)
        h = C.c_void_p()
        _raise(N.load().paes_cuda_batch_plan_create(direction, a[1], b[1], c[1], rks, self.n, int(bool(pad)), device,
                                                    C.byref(h)))
        self._h = h

    def run(self, d_in: int, d_out: int, stream: int = 0):
        """One launch; thread-safe (each call has its own output lengths)."""
        import numpy as np

        olens = np.zeros(max(self.n, 1), dtype=np.uint64)
        _raise(N.load().paes_cuda_batch_plan_run(self._h, d_in, d_out, olens.ctypes.data_as(C.POINTER(C.c_uint64)),
                                                 stream or None))
        return olens[: self.n].tolist()

    def run_async(self, d_in: int, d_out: int, d_out_lens: int, stream: int = 0) -> None:
        """Queued run (paes_cuda_batch_plan_run_async): no sync, graph-capturable;
        the n uint64 words at ``d_out_lens`` receive the output lengths
        (``BAD_PAD`` for a malformed trailer) when the kernel has run."""
        _raise(N.load().paes_cuda_batch_plan_run_async(self._h, d_in, d_out, d_out_lens, stream or None))

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            N.load().paes_cuda_batch_plan_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def sweep(seed: int, size: int) -> bytes:
    """generate_sweep_file (bench.cpp:109-125) into memory."""
    out = C.create_string_buffer(max(size, 1))
    _raise(N.load().paes_cuda_sweep(seed, size, out))
    return out.raw[:size]


def sweep_into(seed: int, size: int, ptr: int) -> None:
    _raise(N.load().paes_cuda_sweep(seed, size, ptr))


def batch_lengths(seed: int, n: int) -> List[int]:
    arr = (C.c_uint64 * max(n, 1))()
    _raise(N.load().paes_cuda_batch_lengths(seed, n, arr))
    return list(arr[:n])


def counter_fill(seed: int, offset: int, size: int) -> bytes:
    out = C.create_string_buffer(max(size, 1))
    _raise(N.load().paes_cuda_counter_fill(seed, offset, size, out))
    return out.raw[:size]


def counter_fill_device(seed: int, offset: int, size: int, d_out: int, device: int = 0, stream: int = 0) -> None:
    _raise(N.load().paes_cuda_counter_fill_device(seed, offset, size, d_out, device, stream or None))


def checksum(data, base_word: int = 0) -> int:
    src = _InBuf(data)
    out = C.c_uint64()
    _raise(N.load().paes_cuda_checksum(src.ptr, src.n, base_word, C.byref(out)))
    return out.value


def checksum_device(d_buf: int, nbytes: int, base_word: int = 0, device: int = 0, stream: int = 0) -> int:
    out = C.c_uint64()
    _raise(N.load().paes_cuda_checksum_device(d_buf, nbytes, base_word, C.byref(out), device, stream or None))
    return out.value


def count_mismatch_device(d_a: int, d_b: int, nbytes: int, device: int = 0, stream: int = 0) -> int:
    out = C.c_uint64()
    _raise(N.load().paes_cuda_count_mismatch_device(d_a, d_b, nbytes, C.byref(out), device, stream or None))
    return out.value


def launch_count() -> int:
    return int(N.load().paes_cuda_launch_count())


def version() -> str:
    return N.load().paes_cuda_version().decode()
