"""Device-resident throughput of paes_cuda_ecb_device at pointer offsets
0 / 1 / 4 / 8 (the ALIGNED=false instantiation handles any offset).
One JSON line; CUDA-event timing, 1 GiB, best of 5."""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

from paper_1403_7295_b200 import paes  # noqa: E402

n = 1 << 30
rk = paes.round_keys(bytes(range(16)))
a = torch.empty(n + 64, dtype=torch.uint8, device="cuda")
b = torch.empty(n + 64, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()
res = {}
for off in (0, 1, 4, 8):
    fn = lambda: paes.ecb_device(0, a.data_ptr() + off, b.data_ptr() + off, n, rk, 0, s.cuda_stream)  # noqa: E731
    fn()
    best = 0.0
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        fn()
        e1.record(s)
        e1.synchronize()
        best = max(best, n / (e0.elapsed_time(e1) / 1e3) / 1e9)
    res[f"off{off}_gbs"] = round(best, 1)
print(json.dumps(res))
