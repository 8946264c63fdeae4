"""Device-resident A/B of the bulk kernel between library builds: queued
paes_cuda_ecb_device launches over 4 GiB (> L2), encrypt then decrypt, 10
launches between one event pair, best of 3 pairs.  Run once per build
(PAES_CUDA_LIB=<variant>).  One JSON line.
    python scripts/kernel_ab_probe.py"""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

from paper_1403_7295_b200 import paes  # noqa: E402

n = 4 << 30
a = torch.empty(n + 16, dtype=torch.uint8, device="cuda")
b = torch.empty(n + 16, dtype=torch.uint8, device="cuda")
paes.counter_fill_device(7, 0, n, a.data_ptr())
rk = paes.round_keys(bytes(range(16)))
s = torch.cuda.current_stream().cuda_stream
res = {}
for d, (src, dst) in ((0, (a, b)), (1, (b, a))):
    best = 0.0
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        paes.ecb_device(d, src.data_ptr(), dst.data_ptr(), n, rk, 0, s)
        e0.record()
        for _ in range(10):
            paes.ecb_device(d, src.data_ptr(), dst.data_ptr(), n, rk, 0, s)
        e1.record()
        e1.synchronize()
        best = max(best, 10 * n / (e0.elapsed_time(e1) / 1e3) / 1e9)
    res["encrypt" if d == 0 else "decrypt"] = round(best, 1)
print(json.dumps({"lib": os.environ.get("PAES_CUDA_LIB", "in-tree"), **res}))
