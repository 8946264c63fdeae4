"""Host-address alignment vs pinned copy throughput: paes_cuda_chunk at page-aligned and misaligned offsets, and the host batch with 16-byte vs 4 KiB message alignment."""
import ctypes as C, json, os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_1403_7295_b200 import _native as N, paes
L = N.load(); paes.set_zero_copy_max(0)
n = 2 << 30
host = torch.empty(n + 8192, dtype=torch.uint8, pin_memory=True)
hout = torch.empty(n + 8192, dtype=torch.uint8, pin_memory=True)
rk = paes.round_keys(bytes(16))
def best(fn):
    fn(); b = 0
    for _ in range(3):
        t = time.perf_counter(); fn(); b = max(b, n / (time.perf_counter() - t) / 1e9)
    return round(b, 2)
res = {}
for off in (0, 16, 4096 + 48):
    res[f"chunk_off{off}"] = best(lambda: L.paes_cuda_chunk(0, host.data_ptr() + off, n - 8192, 0, rk, hout.data_ptr() + off, C.byref(C.c_uint64()), 1))
lens = paes.batch_lengths(4, 4096)
for align in (16, 4096):
    in_off, out_off, oi, oo = [], [], 0, 0
    keep = []
    for Lm in lens:
        if oo + Lm + 4096 + 16 > n: break
        in_off.append(oi); out_off.append(oo); keep.append(Lm)
        oi += (Lm + align - 1) // align * align
        oo += ((Lm // 16 + 1) * 16 + align - 1) // align * align
    rks = b"".join(paes.round_keys(bytes([i % 256] * 16)) for i in range(len(keep)))
    tot = sum(keep)
    def fn():
        paes.ecb_batch_host(0, host.data_ptr(), hout.data_ptr(), in_off, out_off, keep, rks, True)
    fn(); b = 0
    for _ in range(3):
        t = time.perf_counter(); fn(); b = max(b, tot / (time.perf_counter() - t) / 1e9)
    res[f"batch_align{align}"] = round(b, 2)
print(json.dumps(res))
