"""Pinned host e2e (paes_cuda_chunk, in place, encrypt, final) over input size
x ring piece size, zero-copy route off, 3 streams; plus the default route
(zero-copy up to paes.DEFAULT_ZERO_COPY_MAX).  One JSON line per cell, GB/s = input bytes / wall
time, best of 3.
    python scripts/ring_piece_sweep.py [sizes_mib=64,256,1024,4096] [pieces_mib=4,8,16,32,64] [streams=3]"""
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

from paper_1403_7295_b200 import _native as N  # noqa: E402
from paper_1403_7295_b200 import paes  # noqa: E402

MiB = 1 << 20
sizes = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "64,256,1024,4096").split(",")]
pieces = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "4,8,16,32,64").split(",")]
streams = [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "3").split(",")]
L = N.load()
rk = paes.round_keys(bytes(16))
olen = C.c_uint64()
host = torch.empty(max(sizes) * MiB + 32, dtype=torch.uint8, pin_memory=True)
host.fill_(7)


def best_of(n, reps=3):
    assert L.paes_cuda_chunk(0, host.data_ptr(), n, 1, rk, host.data_ptr(), C.byref(olen), 1) == 0
    b = 0.0
    for _ in range(reps):
        t = time.perf_counter()
        assert L.paes_cuda_chunk(0, host.data_ptr(), n, 1, rk, host.data_ptr(), C.byref(olen), 1) == 0
        b = max(b, n / (time.perf_counter() - t) / 1e9)
    return round(b, 2)


for size in sizes:
    n = size * MiB
    paes.set_pipeline(256 * MiB, 3)
    paes.set_zero_copy_max(paes.DEFAULT_ZERO_COPY_MAX)
    row = {"size_mib": size, "default": best_of(n)}
    paes.set_zero_copy_max(0)
    row["ring_policy"] = best_of(n)  # the library's own piece size for this length
    for p in pieces:
        for S in streams:
            paes.set_pipeline(p * MiB, S)
            row[f"ring_{p}" + (f"x{S}" if len(streams) > 1 else "")] = best_of(n)
    print(json.dumps(row), flush=True)
paes.set_pipeline(256 * MiB, 3)
paes.set_zero_copy_max(paes.DEFAULT_ZERO_COPY_MAX)
