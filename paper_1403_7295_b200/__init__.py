"""paper_1403_7295_b200 -- B200-native AES-128 ECB bulk-encryption engine.

A drop-in for the reference "paes" library's chunked file-encryption hot path
(AES-128 ECB with PKCS#7 always-pad): hand-written sm_100a kernels behind a C
ABI (include/paes_cuda.h, lib/libpaes_cuda.so), with ``paes`` mirroring the
reference's ``_paes`` Python module.  No CPU fallback exists.
"""
from . import paes  # noqa: F401
from .paes import (DECRYPT, ENCRYPT, GpuError, IoError, PaddingError, WorkerError, decrypt_bytes,  # noqa: F401
                   decrypt_chunk, decrypt_ecb, decrypt_file, encrypt_bytes, encrypt_chunk, encrypt_ecb, encrypt_file,
                   expand_key, plan_chunks, round_keys)

__all__ = ["paes"]
