"""Same-process A/B of the ring slot size (64 MiB vs 256 MiB, 3 streams) on
the paths that use the pinned host slots: pageable 1 GiB chunk calls and
file->file jobs (warm, previous output removed).  One JSON line."""
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402

from paper_1403_7295_b200 import _native as N  # noqa: E402
from paper_1403_7295_b200 import paes  # noqa: E402

L = N.load()
rk = paes.round_keys(bytes(16))
n = 1 << 30
src = np.tile(np.frombuffer(os.urandom(1 << 20), dtype=np.uint8), n >> 20)
dst = np.empty(n + 16, dtype=np.uint8)
fin, fout = "/dev/shm/paes_slot_in", "/dev/shm/paes_slot_out"
src[: 1 << 30].tofile(fin)
key = bytes(range(16))
res = {}
for rep in range(3):
    for slot in (64, 256):
        paes.set_pipeline(slot << 20, 3)
        olen = C.c_uint64()
        L.paes_cuda_chunk(0, src.ctypes.data, n, 1, rk, dst.ctypes.data, C.byref(olen), 1)  # warm this shape
        t = time.perf_counter()
        for _ in range(3):
            L.paes_cuda_chunk(0, src.ctypes.data, n, 1, rk, dst.ctypes.data, C.byref(olen), 1)
        res.setdefault(f"pageable_1GiB_slot{slot}", []).append(round(3 * n / (time.perf_counter() - t) / 1e9, 2))
        paes.encrypt_file(fin, fout, key)
        os.unlink(fout)
        o = paes.encrypt_file(fin, fout, key)
        os.unlink(fout)
        res.setdefault(f"file_1GiB_slot{slot}", []).append(round(n / o["seconds"] / 1e9, 2))
os.unlink(fin)
paes.set_pipeline(256 << 20, 3)
print(json.dumps(res))
