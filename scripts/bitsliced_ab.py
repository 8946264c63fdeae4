"""A/B of the two encrypt kernels the north_star names: T-table (shared
memory, LDS-bound) vs bitsliced (LOP3, ALU-bound).  8 GiB device-resident,
same key, outputs compared; prints one JSON line.  Profile both with
    ncu --set full -k regex:"ecb_kernel|ecb_bitsliced" -s 2 -c 2 python scripts/bitsliced_ab.py --profile
"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

from paper_1403_7295_b200 import _native as N  # noqa: E402
from paper_1403_7295_b200 import paes  # noqa: E402

profile = "--profile" in sys.argv
from paper_1403_7295_b200 import build as B  # noqa: E402

BS = C.CDLL(B.BITSLICED_AB)
BS.paes_bitsliced_ab_ecb.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p]
n = (1 << 30) if profile else (8 << 30)
rk = paes.round_keys(paes.sweep(3, 16))
pt = torch.empty(n, dtype=torch.uint8, device="cuda")
a = torch.empty(n, dtype=torch.uint8, device="cuda")
b = torch.empty(n, dtype=torch.uint8, device="cuda")
paes.counter_fill_device(3, 0, n, pt.data_ptr())
s = torch.cuda.Stream()


def ttable():
    paes.ecb_device(0, pt.data_ptr(), a.data_ptr(), n, rk, 0, s.cuda_stream)


def bitsliced():
    rc = BS.paes_bitsliced_ab_ecb(pt.data_ptr(), b.data_ptr(), n, rk, s.cuda_stream)
    assert rc == 0, rc


res = {"bytes": n}
for name, fn in [("ttable", ttable), ("bitsliced", bitsliced)]:
    reps = 1 if profile else 5
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    res[name + "_gbs"] = round(n * reps / (e0.elapsed_time(e1) / 1e3) / 1e9, 1)
res["identical"] = paes.count_mismatch_device(a.data_ptr(), b.data_ptr(), n) == 0
print(json.dumps(res))
