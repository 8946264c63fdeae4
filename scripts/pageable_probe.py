"""Host-pointer throughput with PAGEABLE buffers (what std::vector / Python
bytes callers pass) vs pinned, through paes_cuda_chunk."""
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1403_7295_b200 import _native as N  # noqa: E402
from paper_1403_7295_b200 import paes  # noqa: E402

L = N.load()
rk = paes.round_keys(bytes(16))
res = {}
for n in (64 << 20, 1 << 30):
    a = np.frombuffer(os.urandom(1 << 20), dtype=np.uint8)
    src = np.tile(a, n >> 20)
    dst = np.empty(n + 16, dtype=np.uint8)
    olen = C.c_uint64()
    for label, s_ptr, d_ptr in [("pageable", src.ctypes.data, dst.ctypes.data)]:
        L.paes_cuda_chunk(0, s_ptr, n, 1, rk, d_ptr, C.byref(olen), 1)
        t = time.perf_counter()
        for _ in range(3):
            assert L.paes_cuda_chunk(0, s_ptr, n, 1, rk, d_ptr, C.byref(olen), 1) == 0
        res[f"{label}_{n >> 20}MiB_gbs"] = round(3 * n / (time.perf_counter() - t) / 1e9, 2)
    hs = torch.empty(n + 32, dtype=torch.uint8, pin_memory=True)
    hd = torch.empty(n + 32, dtype=torch.uint8, pin_memory=True)
    L.paes_cuda_chunk(0, hs.data_ptr(), n, 1, rk, hd.data_ptr(), C.byref(olen), 1)
    t = time.perf_counter()
    for _ in range(3):
        assert L.paes_cuda_chunk(0, hs.data_ptr(), n, 1, rk, hd.data_ptr(), C.byref(olen), 1) == 0
    res[f"pinned_{n >> 20}MiB_gbs"] = round(3 * n / (time.perf_counter() - t) / 1e9, 2)
print(json.dumps(res))
