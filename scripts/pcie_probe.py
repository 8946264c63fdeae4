"""PCIe ceiling + host-pipeline tuning probe (run on the GPU box).

Measures pinned H2D, D2H and concurrent H2D+D2H copy bandwidth with plain
cudaMemcpyAsync (torch), then the engine's host-pointer path (paes_cuda_chunk)
over a grid of staging chunk sizes x stream counts.  Prints one JSON line.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

from paper_1403_7295_b200 import _native as N  # noqa: E402
from paper_1403_7295_b200 import paes  # noqa: E402

GiB = 1 << 30
MiB = 1 << 20


def bw_copy(n=4 * GiB, reps=3):
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    res = {}
    for name in ("h2d", "d2h", "both"):
        best = 0
        for _ in range(reps):
            torch.cuda.synchronize()
            t = time.perf_counter()
            if name in ("h2d", "both"):
                with torch.cuda.stream(s1):
                    d.copy_(h, non_blocking=True)
            if name in ("d2h", "both"):
                with torch.cuda.stream(s2):
                    h2.copy_(d2, non_blocking=True)
            torch.cuda.synchronize()
            el = time.perf_counter() - t
            best = max(best, n / el / 1e9)
        res[name] = round(best, 2)
    del h, h2, d, d2
    return res


def e2e_grid(n=8 * GiB):
    host = torch.empty(n + 32, dtype=torch.uint8, pin_memory=True)
    host[:n].fill_(7)
    rk = paes.round_keys(bytes(16))
    L = N.load()
    olen = C.c_uint64()
    out = {}
    for chunk in (8, 16, 32, 64, 128):
        for streams in (2, 3, 4, 6):
            paes.set_pipeline(chunk * MiB, streams)
            L.paes_cuda_chunk(0, host.data_ptr(), n, 1, rk, host.data_ptr(), C.byref(olen), 1)  # warm
            t = time.perf_counter()
            for _ in range(2):
                rc = L.paes_cuda_chunk(0, host.data_ptr(), n, 1, rk, host.data_ptr(), C.byref(olen), 1)
                assert rc == 0, N.last_error()
            el = (time.perf_counter() - t) / 2
            out[f"{chunk}MiBx{streams}"] = round(n / el / 1e9, 2)
    paes.set_pipeline(256 * MiB, 3)  # the library default
    return out


if __name__ == "__main__":
    r = {"copy_gbs": bw_copy()}
    r["e2e_gbs"] = e2e_grid()
    print(json.dumps(r))
