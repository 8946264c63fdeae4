"""paes_cuda_batch_host (config-5 layout, pinned host) against paes_cuda_chunk
on the same total bytes, across pipeline shapes (piece bytes x streams).
One JSON line; GB/s = input bytes / wall time, best of 3."""
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

from paper_1403_7295_b200 import _native as N  # noqa: E402
from paper_1403_7295_b200 import paes  # noqa: E402

lens = paes.batch_lengths(4, 4096)
in_off, out_off, oi, oo = [], [], 0, 0
for L in lens:
    in_off.append(oi)
    out_off.append(oo)
    oi += (L + 15) // 16 * 16
    oo += (L // 16 + 1) * 16
rks = b"".join(paes.round_keys(bytes([i % 256] * 16)) for i in range(len(lens)))
host = torch.empty(oi + 16, dtype=torch.uint8, pin_memory=True)
hout = torch.empty(oo + 16, dtype=torch.uint8, pin_memory=True)
rk = paes.round_keys(bytes(16))
L = N.load()
paes.set_zero_copy_max(0)
res = {"total_bytes": oi, "rows": []}
for piece, streams in [(32 << 20, 3), (64 << 20, 3), (128 << 20, 3), (64 << 20, 4), (128 << 20, 4), (256 << 20, 3)]:
    paes.set_pipeline(piece, streams)
    row = {"piece_mib": piece >> 20, "streams": streams}
    for name, fn in [("batch_host", lambda: paes.ecb_batch_host(0, host.data_ptr(), hout.data_ptr(), in_off, out_off,
                                                                  lens, rks, True)),
                     ("chunk", lambda: L.paes_cuda_chunk(0, host.data_ptr(), oi, 0, rk, hout.data_ptr(),
                                                         C.byref(C.c_uint64()), 1))]:
        fn()
        best = 0.0
        for _ in range(3):
            t = time.perf_counter()
            fn()
            best = max(best, oi / (time.perf_counter() - t) / 1e9)
        row[name + "_gbs"] = round(best, 2)
    res["rows"].append(row)
paes.set_pipeline(256 << 20, 3)  # the library default
print(json.dumps(res))
