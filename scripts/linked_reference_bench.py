"""The reference's own code paths with ONLY aes.cpp swapped for the engine
(oracle/_ref/linked/_paes*.so: unmodified paes_module.cpp + chunk/exec/bench/
report.cpp linked against lib/libpaes_aes_b200.so), next to the same paths
in the reference's all-CPU build (oracle/_ref/libpaes_ref.so, as bench.py's
reference arm) -- what a user gets from the link-level drop-in alone.

    PYTHONPATH=oracle/_ref/linked python scripts/linked_reference_bench.py [--gib 4]

Rows (GB/s of input, 1 warm + 3 timed reps, reject-outliers-free mean):
  run_job encrypt file -> file on /dev/shm, strategies sequential / threads W
  (JobOutcome.seconds, exec.cpp:143-202), and encrypt_bytes / decrypt_bytes
  (paes_module.cpp:84-93: encrypt_chunk -> pad_final copy -> encrypt_ecb).
Prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref", "linked"))
sys.path.insert(0, ROOT)

import _paes  # noqa: E402  (the linked reference module)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gib", type=float, default=4.0)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    assert "linked" in _paes.__file__, _paes.__file__
    from paper_1403_7295_b200 import paes

    n = int(args.gib * (1 << 30)) + 7
    key = paes.sweep(2, 16)
    data = paes.sweep(2, n)
    rows = {}
    d = tempfile.mkdtemp(dir="/dev/shm" if os.path.isdir("/dev/shm") else None)
    src, enc = os.path.join(d, "in.bin"), os.path.join(d, "out.enc")
    with open(src, "wb") as f:
        f.write(data)
    try:
        for strategy, w in (("sequential", 1), ("threads", 4), ("threads", 16)):
            secs = []
            for i in range(args.reps + 1):
                o = _paes.encrypt_file(src, enc, key, w, strategy)
                if i:
                    secs.append(o["seconds"])
            rows[f"run_job_{strategy}_w{w}_gbs"] = round(n / (sum(secs) / len(secs)) / 1e9, 3)
            rows[f"run_job_{strategy}_w{w}_seconds"] = [round(s, 4) for s in secs]
        ok_file = open(enc, "rb").read() == paes.encrypt_bytes(data, key)
        secs = []
        for i in range(args.reps + 1):
            t = time.perf_counter()
            ct = _paes.encrypt_bytes(data, key)
            if i:
                secs.append(time.perf_counter() - t)
        rows["encrypt_bytes_gbs"] = round(n / (sum(secs) / len(secs)) / 1e9, 3)
        secs = []
        for i in range(args.reps + 1):
            t = time.perf_counter()
            pt = _paes.decrypt_bytes(ct, key)
            if i:
                secs.append(time.perf_counter() - t)
        rows["decrypt_bytes_gbs"] = round(len(ct) / (sum(secs) / len(secs)) / 1e9, 3)
        ok_bytes = pt == data and ct == paes.encrypt_bytes(data, key)
    finally:
        for p in (src, enc):
            if os.path.exists(p):
                os.unlink(p)
        os.rmdir(d)
    print(json.dumps({"bytes": n, "module": _paes.__file__, "parity": "ok" if ok_file and ok_bytes else "MISMATCH",
                      "launches": paes.launch_count(), **rows}))


if __name__ == "__main__":
    main()
