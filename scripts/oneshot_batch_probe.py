"""Wall time per call of the one-shot paes_cuda_ecb_batch (config-5 layout, device buffers): queued back to back and synchronised."""
import os, sys, time, json
sys.path.insert(0, os.getcwd())
import torch
from paper_1403_7295_b200 import paes
n = 4096
lens = paes.batch_lengths(4, n)
in_off, out_off, oi, oo = [], [], 0, 0
for L in lens:
    in_off.append(oi); out_off.append(oo); oi += L; oo += L + 16
rks = b"".join(paes.round_keys(bytes([i % 256] * 16)) for i in range(n))
src = torch.zeros(oi + 16, dtype=torch.uint8, device="cuda")
dst = torch.zeros(oo + 16, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
res = {}
for rep in range(3):
    for _ in range(3):
        paes.ecb_batch(0, src.data_ptr(), dst.data_ptr(), in_off, out_off, lens, rks, True, 0, s.cuda_stream)
    s.synchronize()
    t = time.perf_counter()
    for _ in range(10):
        paes.ecb_batch(0, src.data_ptr(), dst.data_ptr(), in_off, out_off, lens, rks, True, 0, s.cuda_stream)
    s.synchronize()
    res[f"rep{rep}_ms_per_call"] = round((time.perf_counter() - t) / 10 * 1e3, 3)
t = time.perf_counter()
for _ in range(10):
    paes.ecb_batch(0, src.data_ptr(), dst.data_ptr(), in_off, out_off, lens, rks, True, 0, s.cuda_stream)
    s.synchronize()
res["synced_ms_per_call"] = round((time.perf_counter() - t) / 10 * 1e3, 3)
print(json.dumps(res))
