"""Pinned e2e (paes_cuda_chunk, in place, encrypt, final) at 32-512 MiB with the
zero-copy limit raised over the size (one 32-CTA zero-copy kernel) and at 0
(the copy ring), alternating, best of R.  One JSON line.
    python scripts/zc_vs_ring_probe.py [sizes_mib=32,48,64,96,128,256,512] [reps=5]"""
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
sizes = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "32,48,64,96,128,256,512").split(",")]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
host = torch.empty(max(sizes) * MiB + 32, dtype=torch.uint8, pin_memory=True)
host.fill_(7)
L = N.load()
rk = paes.round_keys(bytes(16))
olen = C.c_uint64()
res = {}
for mib in sizes:
    n = mib * MiB
    row = {}
    for route, zc in (("zero_copy", 1 << 40), ("ring", 0)):
        paes.set_zero_copy_max(zc)
        assert L.paes_cuda_chunk(0, host.data_ptr(), n, 1, rk, host.data_ptr(), C.byref(olen), 1) == 0
        best = 0.0
        for _ in range(reps):
            t = time.perf_counter()
            assert L.paes_cuda_chunk(0, host.data_ptr(), n, 1, rk, host.data_ptr(), C.byref(olen), 1) == 0
            best = max(best, n / (time.perf_counter() - t) / 1e9)
        row[route] = round(best, 2)
    res[f"{mib}MiB"] = row
paes.set_zero_copy_max(paes.DEFAULT_ZERO_COPY_MAX)
print(json.dumps(res))
