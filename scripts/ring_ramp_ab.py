"""E2E through paes_cuda_chunk on pinned buffers (the pinned ring) at the
configs' sizes.  Round 2 used it for an A/B of a ramped piece schedule
(C/8, C/4, C/2 at both ends, PAES_RING_RAMP=1 in that build): no gain, not
adopted (profiles/r02_ring_ramp_ab.jsonl).
    python scripts/ring_ramp_ab.py
Prints one JSON line: median GB/s of 7 calls (after 2 warm) per size and direction."""
import ctypes as C
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1403_7295_b200 import _native as N  # noqa: E402
from paper_1403_7295_b200 import paes  # noqa: E402

L = N.load()
rk = paes.round_keys(bytes(range(16)))
res = {"ramp": os.environ.get("PAES_RING_RAMP", "1")}
for n in (64 << 20, (256 << 20) + 7, 1 << 30, 4 << 30):
    src = torch.randint(0, 256, (n + 32,), dtype=torch.uint8).pin_memory()
    dst = torch.empty(n + 32, dtype=torch.uint8).pin_memory()
    back = torch.empty(n + 32, dtype=torch.uint8).pin_memory()
    olen = C.c_uint64()
    out = {}
    for name, (d, a, b, ln) in {"enc": (0, src, dst, n), "dec": (1, dst, back, (n // 16 + 1) * 16)}.items():
        ts = []
        for i in range(9):
            t = time.perf_counter()
            rc = L.paes_cuda_chunk(d, a.data_ptr(), ln, 1, rk, b.data_ptr(), C.byref(olen), 1)
            assert rc == 0, N.last_error()
            if i >= 2:
                ts.append(time.perf_counter() - t)
        out[name] = round(ln / statistics.median(ts) / 1e9, 2)
    assert torch.equal(back[:n], src[:n])
    res[n] = out
    del src, dst, back
print(json.dumps(res))
