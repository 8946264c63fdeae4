"""Device-resident A/B of the bulk kernel between library builds: queued
paes_cuda_ecb_device launches, encrypt then decrypt, at 4 GiB (> L2) and at
64 MiB / 16 MiB rotating over buffer pairs (cold inputs), best of 3 event
pairs.  Run once per build
(PAES_CUDA_LIB=<variant>).  One JSON line.
    python scripts/kernel_ab_probe.py"""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

from paper_1403_7295_b200 import paes  # noqa: E402

rk = paes.round_keys(bytes(range(16)))
s = torch.cuda.current_stream().cuda_stream
res = {}
# 4 GiB (one pair, > L2) and 64 MiB / 16 MiB (rotating over pairs so every
# launch reads cold data, as bench.py config 1 does), 10..40 queued launches
for n, pairs in ((4 << 30, 1), (64 << 20, 4), (16 << 20, 16)):
    bufs = [(torch.empty(n + 16, dtype=torch.uint8, device="cuda"), torch.empty(n + 16, dtype=torch.uint8, device="cuda"))
            for _ in range(pairs)]
    for a, _ in bufs:
        paes.counter_fill_device(7, 0, n, a.data_ptr())
    K = 10 if n >= (1 << 30) else 40
    for d in (0, 1):
        best = 0.0
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            paes.ecb_device(d, bufs[0][0].data_ptr(), bufs[0][1].data_ptr(), n, rk, 0, s)
            e0.record()
            for i in range(K):
                src, dst = bufs[i % pairs] if d == 0 else bufs[i % pairs][::-1]
                paes.ecb_device(d, src.data_ptr(), dst.data_ptr(), n, rk, 0, s)
            e1.record()
            e1.synchronize()
            best = max(best, K * n / (e0.elapsed_time(e1) / 1e3) / 1e9)
        res[f"{'enc' if d == 0 else 'dec'}_{n >> 20}MiB"] = round(best, 1)
    del bufs
    torch.cuda.empty_cache()
print(json.dumps({"lib": os.environ.get("PAES_CUDA_LIB", "in-tree"), **res}))
