"""Per-call cost of paes_cuda_batch_host on 4096 tiny messages: host-side preparation (validation, grouping, key words) dominates."""
import os, sys, time, json
sys.path.insert(0, os.getcwd())
import torch
from paper_1403_7295_b200 import paes
n = 4096
lens = [16] * n
offs = [32 * i for i in range(n)]
rks = b"".join(paes.round_keys(bytes([i % 256] * 16)) for i in range(n))
h = torch.zeros(32 * n + 64, dtype=torch.uint8, pin_memory=True)
o = torch.zeros(32 * n + 64, dtype=torch.uint8, pin_memory=True)
res = {}
for d in (0, 1):
    paes.ecb_batch_host(d, h.data_ptr(), o.data_ptr(), offs, offs, lens, rks, False)
    t = time.perf_counter()
    for _ in range(20):
        paes.ecb_batch_host(d, h.data_ptr(), o.data_ptr(), offs, offs, lens, rks, False)
    res["dir%d_ms" % d] = round((time.perf_counter() - t) / 20 * 1e3, 3)
import numpy as np
a = np.array(offs, dtype=np.uint64)
t = time.perf_counter()
for _ in range(20):
    paes._u64_array(offs); paes._u64_array(lens)
res["python_arrays_ms"] = round((time.perf_counter() - t) / 20 * 1e3, 3)
print(json.dumps(res))
