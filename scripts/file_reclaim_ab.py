"""A/B of the deferred reclaim of a replaced output file (abi_file.cu
ReplacedOutput): run_job on /dev/shm, each rep renaming over the previous
output, with PAES_FILE_ASYNC_RECLAIM=0 (old pages freed inside rename) and 1
(freed on a detached thread).  Prints JobOutcome.seconds per rep, the wall
clock of the whole back-to-back loop (so a reaper that merely moved its cost
into the next job would show), and checks the output digest every time.

    python scripts/file_reclaim_ab.py [--size BYTES] [--reps R] [--dir /dev/shm]
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_1403_7295_b200 import paes  # noqa: E402


def sha(path):
    h = hashlib.sha256()
    with open(path, "rb") as f:
        while True:
            b = f.read(64 << 20)
            if not b:
                break
            h.update(b)
    return h.hexdigest()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=(4 << 30) + 7)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--dir", default="/dev/shm")
    ap.add_argument("--modes", default="0,1", help="values of the switch to compare")
    ap.add_argument("--env", default="PAES_FILE_ASYNC_RECLAIM",
                    help="the 0/1 switch to A/B (also PAES_FILE_PREALLOC: fallocate thread ahead of the mapped writers)")
    args = ap.parse_args()
    key = bytes(range(16))
    src = os.path.join(args.dir, f"paes_ab_in_{os.getpid()}.bin")
    ct = os.path.join(args.dir, f"paes_ab_ct_{os.getpid()}.bin")
    pt = os.path.join(args.dir, f"paes_ab_pt_{os.getpid()}.bin")
    rng = np.random.default_rng(3)
    with open(src, "wb") as f:
        left = args.size
        while left:
            n = min(left, 256 << 20)
            f.write(rng.integers(0, 256, n, dtype=np.uint8).tobytes())
            left -= n
    res = {"size": args.size, "dir": args.dir, "reps": args.reps, "switch": args.env}
    try:
        paes.encrypt_file(src, ct, key, workers=1)  # warm: context, ring, page cache
        want_ct, want_pt = sha(ct), sha(src)
        modes = tuple(args.modes.split(","))
        for order in (modes, modes[::-1]):  # both orders: no drift credit
            for mode in order:
                os.environ[args.env] = mode
                for name, fn, out, want in (("enc", lambda: paes.encrypt_file(src, ct, key, workers=1), ct, want_ct),
                                            ("dec", lambda: paes.decrypt_file(ct, pt, key, workers=1), pt, want_pt)):
                    fn()
                    t = time.perf_counter()
                    secs = [fn()["seconds"] for _ in range(args.reps)]
                    wall = time.perf_counter() - t
                    time.sleep(0.5)  # let a reaper finish before the digest read
                    ok = sha(out) == want
                    n = args.size
                    res.setdefault(f"{args.env}={mode}", []).append(
                        {"op": name, "job_seconds": [round(x, 4) for x in secs],
                         "gbs_job_median": round(n / sorted(secs)[len(secs) // 2] / 1e9, 3),
                         "gbs_loop_wall": round(n * args.reps / wall / 1e9, 3), "parity": "ok" if ok else "MISMATCH"})
    finally:
        for p in (src, ct, pt):
            if os.path.exists(p):
                os.unlink(p)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
