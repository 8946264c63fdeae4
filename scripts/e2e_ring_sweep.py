"""The bench's e2e call (paes_cuda_chunk, in place on one pinned 64 GiB host
buffer, zero-copy off since the range is > 128 MiB) over ring shapes: piece
bytes x streams.  One JSON line, GB/s = input bytes / wall time, best of 2."""
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

from paper_1403_7295_b200 import _native as N  # noqa: E402
from paper_1403_7295_b200 import paes  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else (64 << 30)
host = torch.empty(n + 32, dtype=torch.uint8, pin_memory=True)
host[: 1 << 20].fill_(7)
L = N.load()
rk = paes.round_keys(bytes(16))
olen = C.c_uint64()
res = {"bytes": n, "rows": []}
for piece, streams in [(64, 3), (64, 4), (128, 3), (128, 4), (128, 6), (256, 3), (256, 4)]:
    paes.set_pipeline(piece << 20, streams)
    L.paes_cuda_chunk(0, host.data_ptr(), n, 1, rk, host.data_ptr(), C.byref(olen), 1)
    best = 0.0
    for _ in range(2):
        t = time.perf_counter()
        assert L.paes_cuda_chunk(0, host.data_ptr(), n, 1, rk, host.data_ptr(), C.byref(olen), 1) == 0
        best = max(best, n / (time.perf_counter() - t) / 1e9)
    res["rows"].append({"piece_mib": piece, "streams": streams, "gbs": round(best, 2)})
paes.set_pipeline(256 << 20, 3)  # the library default
print(json.dumps(res))
