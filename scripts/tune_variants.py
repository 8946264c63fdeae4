"""Kernel shape tuning: blocks-per-thread (NB) x CTA threads.

    python scripts/tune_variants.py build        # here (nvcc, no GPU): tune/<NB>_<T>/libpaes_cuda.so
    python scripts/tune_variants.py run          # on the B200: one subprocess per variant, JSON lines

Each variant times the device-resident encrypt and decrypt of 8 GiB (one
launch per step, CUDA events) and checks its ciphertext checksum against the
default build's.
"""
from __future__ import annotations

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
TUNE = os.path.join(ROOT, "tune")
VARIANTS = [(nb, t) for nb in (1, 2, 4) for t in (256, 512, 1024)]


def build_all():
    from concurrent.futures import ThreadPoolExecutor

    from paper_1403_7295_b200 import build as b

    def one(v):
        nb, t = v
        try:
            return b.build(force=True, defines=[f"PAES_NB={nb}", f"PAES_THREADS={t}"],
                           out_lib=os.path.join(TUNE, f"{nb}_{t}", "libpaes_cuda.so"))
        except RuntimeError as e:
            return f"FAILED {v}: {str(e)[:300]}"

    with ThreadPoolExecutor(3) as ex:
        for r in ex.map(one, VARIANTS):
            print(r)


def run_one(lib):
    import torch

    from paper_1403_7295_b200 import _native as N
    from paper_1403_7295_b200 import paes

    N.lib_path = lambda: lib
    n = 8 << 30
    rk = paes.round_keys(paes.sweep(3, 16))
    pt = torch.empty(n, dtype=torch.uint8, device="cuda")
    ct = torch.empty(n + 16, dtype=torch.uint8, device="cuda")
    paes.counter_fill_device(3, 0, n, pt.data_ptr())
    s = torch.cuda.Stream()
    res = {"lib": os.path.relpath(lib, ROOT)}
    for name, fn in [("enc", lambda: paes.chunk_device(0, pt.data_ptr(), n, False, rk, ct.data_ptr(), 0, s.cuda_stream)),
                     ("dec", lambda: paes.ecb_device(1, ct.data_ptr(), pt.data_ptr(), n, rk, 0, s.cuda_stream))]:
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(5):
            fn()
        b.record(s)
        torch.cuda.synchronize()
        res[name + "_gbs"] = round(n * 5 / (a.elapsed_time(b) / 1e3) / 1e9, 1)
        if name == "enc":
            res["ct_checksum"] = paes.checksum_device(ct.data_ptr(), n, 0)
    print(json.dumps(res), flush=True)


def run_all():
    libs = [os.path.join(TUNE, f"{nb}_{t}", "libpaes_cuda.so") for nb, t in VARIANTS]
    for lib in libs:
        if not os.path.exists(lib):
            print(json.dumps({"lib": lib, "error": "not built"}))
            continue
        r = subprocess.run([sys.executable, __file__, "one", lib], capture_output=True, text=True, timeout=600)
        print(r.stdout.strip() or json.dumps({"lib": lib, "error": r.stderr[-500:]}), flush=True)


if __name__ == "__main__":
    cmd = sys.argv[1] if len(sys.argv) > 1 else "run"
    if cmd == "build":
        build_all()
    elif cmd == "one":
        run_one(sys.argv[2])
    else:
        run_all()
