"""Pageable (Python bytes) encrypt_bytes / decrypt_bytes at 16 KiB .. 8 MiB,
single thread, best of R: GB/s and us per call.  Run with PAES_BOUNCE_MAX=0
to push every size onto the staged ring (A/B of the bounce-buffer path).
    python scripts/pageable_small_probe.py [reps=30] [sizes_kib=16,64,256,512,1024,2048,8192]"""
import json
import os
import sys
import time

sys.path.insert(0, os.getcwd())
from paper_1403_7295_b200 import paes  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
key = bytes(range(16))
res = {}
sizes = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "16,64,256,512,1024,2048,8192").split(",")]
for kib in sizes:
    n = kib * 1024 + 7
    data = os.urandom(n)
    ct = paes.encrypt_bytes(data, key)
    assert paes.decrypt_bytes(ct, key) == data
    best_e = best_d = 1e9
    for _ in range(reps):
        t = time.perf_counter()
        paes.encrypt_bytes(data, key)
        best_e = min(best_e, time.perf_counter() - t)
        t = time.perf_counter()
        paes.decrypt_bytes(ct, key)
        best_d = min(best_d, time.perf_counter() - t)
    res[f"{kib}KiB"] = {"enc_us": round(best_e * 1e6, 1), "enc_gbs": round(n / best_e / 1e9, 2),
                        "dec_us": round(best_d * 1e6, 1), "dec_gbs": round(len(ct) / best_d / 1e9, 2)}
print(json.dumps(res))
