"""First-call cost of the file path in a fresh process (what a one-shot CLI
user of run_job sees): JobOutcome.seconds and wall clock of call 1 and call 2,
plus the process's import-to-exit time.

    python scripts/file_cold_probe.py [--size BYTES] [--dir /dev/shm]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

T0 = time.perf_counter()
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_1403_7295_b200 import paes  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=(4 << 30) + 7)
    ap.add_argument("--dir", default="/dev/shm")
    args = ap.parse_args()
    src = os.path.join(args.dir, f"paes_cold_in_{os.getpid()}.bin")
    out = os.path.join(args.dir, f"paes_cold_out_{os.getpid()}.bin")
    rng = np.random.default_rng(5)
    with open(src, "wb") as f:
        left = args.size
        while left:
            n = min(left, 256 << 20)
            f.write(rng.integers(0, 256, n, dtype=np.uint8).tobytes())
            left -= n
    key = bytes(range(16))
    res = {"size": args.size, "import_s": round(time.perf_counter() - T0, 3)}
    try:
        for i in (1, 2, 3):
            t = time.perf_counter()
            r = paes.encrypt_file(src, out, key, workers=1, strategy="gpu")
            res[f"call{i}"] = {"job_s": round(r["seconds"], 4), "wall_s": round(time.perf_counter() - t, 4)}
            os.unlink(out)
    finally:
        for p in (src, out):
            if os.path.exists(p):
                os.unlink(p)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
