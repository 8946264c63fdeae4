"""Where the per-call host cost of the device-pointer API goes (round 2).

    python scripts/host_tax_probe.py

For 1 MiB / 16 MiB / 64 MiB device buffers: queued device GB/s of K calls
between one event pair for (a) paes_cuda_ecb_device, (b) paes_cuda_chunk_device
encrypt with always-pad, (c) chunk_device final decrypt (synchronous trailer
check), each from the C ABI via ctypes with pre-built arguments and through
paes.chunk_device; plus the host wall time per call of each.  Prints JSON.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1403_7295_b200 import _native as N  # noqa: E402
from paper_1403_7295_b200 import paes  # noqa: E402

MiB = 1 << 20


def queued(fn, steps, stream):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t = time.perf_counter()
    a.record(stream)
    for _ in range(steps):
        fn()
    b.record(stream)
    host = time.perf_counter() - t
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps * 1e3, host / steps * 1e6


def main():
    L = N.load()
    s = torch.cuda.Stream()
    sp = C.c_void_p(s.cuda_stream)
    rk = paes.round_keys(bytes(range(16)))
    rkb = (C.c_uint8 * 176).from_buffer_copy(rk)
    olen = C.c_uint64()
    rows = []
    for n in (1 * MiB, 16 * MiB, 64 * MiB):
        x = torch.randint(0, 256, (n + 32,), dtype=torch.uint8, device="cuda")
        y = torch.empty(n + 32, dtype=torch.uint8, device="cuda")
        z = torch.empty(n + 32, dtype=torch.uint8, device="cuda")
        xp, yp, zp = x.data_ptr(), y.data_ptr(), z.data_ptr()
        paes.chunk_device(0, xp, n, True, rk, yp, 0, s.cuda_stream)
        steps = max(20, int(2e9 // n))
        r = {"bytes": n, "steps": steps}
        for name, fn in [
            ("ecb_c", lambda: L.paes_cuda_ecb_device(0, xp, zp, n, rkb, 0, sp)),
            ("chunk_enc_c", lambda: L.paes_cuda_chunk_device(0, xp, n, 1, rkb, zp, C.byref(olen), 0, sp)),
            ("chunk_enc_py", lambda: paes.chunk_device(0, xp, n, True, rk, zp, 0, s.cuda_stream)),
            ("chunk_dec_final_c", lambda: L.paes_cuda_chunk_device(1, yp, n + 16, 1, rkb, zp, C.byref(olen), 0, sp)),
            ("chunk_dec_final_py", lambda: paes.chunk_device(1, yp, n + 16, True, rk, zp, 0, s.cuda_stream)),
        ]:
            dev_us, host_us = queued(fn, steps, s)
            r[name] = {"dev_us": round(dev_us, 2), "gbs": round(n / dev_us / 1e3, 1), "host_us_per_call": round(host_us, 2)}
        rows.append(r)
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
