"""ctypes binding of the C ABI in include/paes_cuda.h (libpaes_cuda.so).

The library is the product: there is no CPU fallback.  If the .so is missing
(not built) every entry point raises ``NativeLibraryMissing``; if no CUDA
device is visible the compute entry points fail with ``ENODEV`` from the
library itself.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

from . import build as _build

ENCRYPT = 0
DECRYPT = 1

OK = 0
EINVAL = -22
EBADMSG = -74
EIO = -5
EWORKER = -1001
ECUDA = -1002
ENODEV = -1003


class NativeLibraryMissing(ImportError):
    pass


class ChunkSpec(C.Structure):
    _fields_ = [("offset", C.c_uint64), ("raw_len", C.c_uint64), ("padded_len", C.c_uint64),
                ("is_final", C.c_int32), ("reserved", C.c_int32)]


class JobOutcome(C.Structure):
    _fields_ = [("bytes_in", C.c_uint64), ("bytes_out", C.c_uint64), ("seconds", C.c_double)]


# (name, restype, argtypes) for every symbol declared in include/paes_cuda.h
_u8p = C.POINTER(C.c_uint8)
_u64 = C.c_uint64
_vp = C.c_void_p
SIGNATURES = [
    ("paes_cuda_last_error", C.c_char_p, []),
    ("paes_cuda_version", C.c_char_p, []),
    ("paes_cuda_device_count", C.c_int, []),
    ("paes_cuda_set_devices", C.c_int, [C.POINTER(C.c_int), C.c_int]),
    ("paes_cuda_set_pipeline", C.c_int, [_u64, C.c_int]),
    ("paes_cuda_set_zero_copy_max", C.c_int, [_u64]),
    ("paes_cuda_expand_key", C.c_int, [_vp, _vp]),
    ("paes_cuda_worker_chunk", C.c_int, [C.c_char_p, _u64, _u64, C.c_int, C.c_int, _vp, C.c_char_p, C.c_int]),
    ("paes_cuda_state_transform", C.c_int, [C.c_int, _vp, _u64, _vp]),
    ("paes_cuda_sbox", C.c_int, [C.c_int, _vp]),
    ("paes_cuda_plan_chunks", C.c_int64, [_u64, C.c_uint32, C.POINTER(ChunkSpec), _u64]),
    ("paes_cuda_plan_decrypt_chunks", C.c_int64, [_u64, C.c_uint32, C.POINTER(ChunkSpec), _u64]),
    ("paes_cuda_auto_shards", C.c_uint32, [_u64, C.c_uint32]),
    ("paes_cuda_pad_final", C.c_int64, [_vp, _u64, _vp]),
    ("paes_cuda_unpad_final", C.c_int64, [_vp, _u64]),
    ("paes_cuda_ecb", C.c_int, [C.c_int, _vp, _vp, _u64, _vp, C.c_int]),
    ("paes_cuda_ecb_device", C.c_int, [C.c_int, _vp, _vp, _u64, _vp, C.c_int, _vp]),
    ("paes_cuda_chunk", C.c_int, [C.c_int, _vp, _u64, C.c_int, _vp, _vp, C.POINTER(_u64), C.c_int]),
    ("paes_cuda_chunk_device", C.c_int, [C.c_int, _vp, _u64, C.c_int, _vp, _vp, C.POINTER(_u64), C.c_int, _vp]),
    ("paes_cuda_chunk_device_async", C.c_int, [C.c_int, _vp, _u64, C.c_int, _vp, _vp, _vp, C.c_int, _vp]),
    ("paes_cuda_ecb_batch", C.c_int, [C.c_int, _vp, _vp, C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_u64), _vp,
                                      C.c_uint32, C.c_int, C.POINTER(_u64), C.c_int, _vp]),
    ("paes_cuda_batch_host", C.c_int, [C.c_int, _vp, _vp, C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_u64), _vp,
                                       C.c_uint32, C.c_int, C.POINTER(_u64), C.c_int]),
    ("paes_cuda_batch_plan_create", C.c_int, [C.c_int, C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_u64), _vp,
                                              C.c_uint32, C.c_int, C.c_int, C.POINTER(_vp)]),
    ("paes_cuda_batch_plan_run", C.c_int, [_vp, _vp, _vp, C.POINTER(_u64), _vp]),
    ("paes_cuda_batch_plan_run_async", C.c_int, [_vp, _vp, _vp, _vp, _vp]),
    ("paes_cuda_batch_plan_destroy", None, [_vp]),
    ("paes_cuda_run_job", C.c_int, [C.c_char_p, C.c_char_p, _vp, C.c_uint32, C.c_int, C.POINTER(JobOutcome)]),
    ("paes_cuda_sweep", C.c_int, [_u64, _u64, _vp]),
    ("paes_cuda_batch_lengths", C.c_int, [_u64, C.c_uint32, C.POINTER(_u64)]),
    ("paes_cuda_counter_fill_device", C.c_int, [_u64, _u64, _u64, _vp, C.c_int, _vp]),
    ("paes_cuda_counter_fill", C.c_int, [_u64, _u64, _u64, _vp]),
    ("paes_cuda_checksum_device", C.c_int, [_vp, _u64, _u64, C.POINTER(_u64), C.c_int, _vp]),
    ("paes_cuda_checksum", C.c_int, [_vp, _u64, _u64, C.POINTER(_u64)]),
    ("paes_cuda_count_mismatch_device", C.c_int, [_vp, _vp, _u64, C.POINTER(_u64), C.c_int, _vp]),
    ("paes_cuda_launch_count", C.c_uint64, []),
]

_lib = None
_lock = threading.Lock()


def lib_path() -> str:
    """The in-tree library, or a variant build named by PAES_CUDA_LIB (sanitizer,
    coverage or tuning builds; there is still no fallback if it is missing)."""
    return os.environ.get("PAES_CUDA_LIB") or _build.LIB


def load(build_if_missing: bool = False):
    """Load libpaes_cuda.so (in-tree).  Raises NativeLibraryMissing if absent."""
    global _lib
    if _lib is not None:  # hot path: no lock once loaded
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = lib_path()
        if not os.path.exists(path):
            if build_if_missing:
                _build.build()
            else:
                raise NativeLibraryMissing(
                    f"{path} is not built; run `python -m paper_1403_7295_b200.build` (no CPU fallback exists)")
        elif "PAES_CUDA_LIB" not in os.environ and _build._stale():
            # never rebuild behind the caller's back (a variant or a copied
            # tree may have skewed mtimes); say that the kernels may be old
            import warnings

            warnings.warn(f"{path} is older than its sources in {_build.CSRC}; rebuild with "
                          "`python -m paper_1403_7295_b200.build` to load the current kernels", RuntimeWarning,
                          stacklevel=2)
        L = C.CDLL(path)
        for name, res, args in SIGNATURES:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
        return L


def last_error() -> str:
    return load().paes_cuda_last_error().decode(errors="replace")
