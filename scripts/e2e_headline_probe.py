"""The bench's e2e call (paes_cuda_chunk, encrypt, final, in place on one
pinned host buffer) at a few sizes, best of R; one JSON line.
    python scripts/e2e_headline_probe.py [sizes_gib=64,4,1] [reps=3]"""
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

from paper_1403_7295_b200 import _native as N  # noqa: E402
from paper_1403_7295_b200 import paes  # noqa: E402

sizes = [float(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "64,4,1").split(",")]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
n_max = int(max(sizes) * (1 << 30))
host = torch.empty(n_max + 32, dtype=torch.uint8, pin_memory=True)
host[: 1 << 20].fill_(7)
L = N.load()
rk = paes.round_keys(bytes(16))
olen = C.c_uint64()
res = {}
for g in sizes:
    n = int(g * (1 << 30))
    assert L.paes_cuda_chunk(0, host.data_ptr(), n, 1, rk, host.data_ptr(), C.byref(olen), 1) == 0
    best = 0.0
    for _ in range(reps):
        t = time.perf_counter()
        assert L.paes_cuda_chunk(0, host.data_ptr(), n, 1, rk, host.data_ptr(), C.byref(olen), 1) == 0
        best = max(best, n / (time.perf_counter() - t) / 1e9)
    res[f"{g:g}GiB"] = round(best, 2)
print(json.dumps(res))
