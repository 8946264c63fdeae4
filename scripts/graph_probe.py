"""Per-call device time of paes.chunk_device issued one by one vs replayed
from a torch-captured CUDA graph (and from a raw cudaStreamBeginCapture
graph via the probe binary), for the PDL trigger placement A/B.
    PAES_CUDA_LIB=<variant .so> python scripts/graph_probe.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1403_7295_b200 import _native as N  # noqa: E402
from paper_1403_7295_b200 import paes  # noqa: E402

s = torch.cuda.Stream()
rk = paes.round_keys(bytes(range(16)))
out = {"lib": N.lib_path()}
for n in (1031, 65543, (1 << 20) + 7, (16 << 20) + 7, 64 << 20):
    x = torch.randint(0, 256, (n + 64,), dtype=torch.uint8, device="cuda")
    y = torch.empty(n + 64, dtype=torch.uint8, device="cuda")
    call = lambda: paes.chunk_device(0, x.data_ptr(), n, True, rk, y.data_ptr(), 0, s.cuda_stream)  # noqa: E731
    K = 200 if n < (16 << 20) else 40
    for _ in range(5):
        call()
    s.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(K):
        call()
    b.record(s)
    b.synchronize()
    q = a.elapsed_time(b) / K * 1e3
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(K):
                call()
    with torch.cuda.stream(s):
        g.replay()  # warm, on s (replay() launches on the current stream)
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        a.record(s)
        g.replay()
        b.record(s)
    b.synchronize()
    gr = a.elapsed_time(b) / K * 1e3
    out[n] = {"queued_us": round(q, 2), "graph_us": round(gr, 2)}
print(json.dumps(out))
