"""Where the pageable e2e (encrypt_bytes on Python bytes) loses time, 4 GiB:
fresh-output allocation / page faults vs the staged ring itself.
    python scripts/pageable_probe2.py"""
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1403_7295_b200 import _native as N  # noqa: E402
from paper_1403_7295_b200 import paes  # noqa: E402

n = 4 << 30
res = {"thp": open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip(),
       "defrag": open("/sys/kernel/mm/transparent_hugepage/defrag").read().strip(), "cpus": os.cpu_count()}
data = np.random.default_rng(0).integers(0, 256, n, dtype=np.uint8).tobytes()
key = bytes(range(16))
rk = paes.round_keys(key)
L = N.load()
paes.encrypt_bytes(data[: 64 << 20], key)


def t(fn, reps=3):
    fn()
    best = 1e9
    for _ in range(reps):
        s = time.perf_counter()
        fn()
        best = min(best, time.perf_counter() - s)
    return round(n / best / 1e9, 2)


res["encrypt_bytes_gbs"] = t(lambda: paes.encrypt_bytes(data, key))
out = bytearray(n + 16)
ob = (C.c_uint8 * (n + 16)).from_buffer(out)
src = C.cast(C.c_char_p(data), C.c_void_p).value
olen = C.c_uint64()
res["chunk_into_prefaulted_gbs"] = t(lambda: L.paes_cuda_chunk(0, src, n, 1, rk, ob, C.byref(olen), 1))
res["fresh_bytes_touch_gbs"] = t(lambda: np.frombuffer(bytearray(n), dtype=np.uint8))  # calloc'd + zero pages
res["np_empty_fill_gbs"] = t(lambda: np.empty(n, dtype=np.uint8).fill(1))
print(json.dumps(res))
