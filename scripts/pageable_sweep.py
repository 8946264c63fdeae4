"""Pageable host e2e (paes_cuda_chunk on numpy buffers, encrypt, final) over
ring stream/slot counts: the staged ring's slots equal the stream count.
One JSON line per (size, streams), GB/s = input bytes / wall time, best of 3.
    python scripts/pageable_sweep.py [sizes_mib=64,256,1024] [streams=3,4,6]"""
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402

from paper_1403_7295_b200 import _native as N  # noqa: E402
from paper_1403_7295_b200 import paes  # noqa: E402

MiB = 1 << 20
sizes = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "64,256,1024").split(",")]
streams = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "3,4,6").split(",")]
L = N.load()
rk = paes.round_keys(bytes(16))
olen = C.c_uint64()
for size in sizes:
    n = size * MiB
    src = np.tile(np.frombuffer(os.urandom(MiB), dtype=np.uint8), size)
    dst = np.zeros(n + 16, dtype=np.uint8)
    row = {"size_mib": size}
    for S in streams:
        paes.set_pipeline(256 * MiB, S)
        assert L.paes_cuda_chunk(0, src.ctypes.data, n, 1, rk, dst.ctypes.data, C.byref(olen), 1) == 0
        best = 0.0
        for _ in range(3):
            t = time.perf_counter()
            assert L.paes_cuda_chunk(0, src.ctypes.data, n, 1, rk, dst.ctypes.data, C.byref(olen), 1) == 0
            best = max(best, n / (time.perf_counter() - t) / 1e9)
        row[f"s{S}"] = round(best, 2)
    print(json.dumps(row), flush=True)
paes.set_pipeline(256 * MiB, 3)
