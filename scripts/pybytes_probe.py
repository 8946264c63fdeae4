"""Wall-clock GB/s of the _paes mirror on 1 GiB of Python bytes (pageable host memory: staged ring + result object)."""
import os, sys, time, json
sys.path.insert(0, os.getcwd())
from paper_1403_7295_b200 import paes
key = bytes(range(16))
data = os.urandom(1 << 30)
paes.encrypt_bytes(data[: 1 << 20], key)
res = {}
for name, fn in (("encrypt_bytes", lambda: paes.encrypt_bytes(data, key)),):
    fn()
    t = time.perf_counter(); ct = fn(); res[name] = round(len(data) / (time.perf_counter() - t) / 1e9, 2)
t = time.perf_counter(); pt = paes.decrypt_bytes(ct, key); res["decrypt_bytes"] = round(len(ct) / (time.perf_counter() - t) / 1e9, 2)
assert pt == data
print(json.dumps({"bytes": len(data), "gbs": res}))
