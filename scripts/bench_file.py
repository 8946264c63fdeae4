"""File -> file throughput: the paper's own measurement (PAPER.md:93-113,
bench.cpp:81-107), reference pthreads strategy vs the engine's "gpu" strategy.

    python scripts/bench_file.py [--size BYTES] [--reps R] [--dir /dev/shm]

Both sides run the full run_job contract (read input file, transform with
always-pad, write the output under a temporary name, rename).  Timing is the
job's own wall clock (JobOutcome.seconds, exec.cpp:144-200) and the mean of
the reps retained by the reference's reject_outliers, as measure_cell does.
Units: GB/s and the paper's Mb/s (10^6 bit/s).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_1403_7295_b200 import paes  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=4 << 30)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--dir", default="/dev/shm")
    args = ap.parse_args()
    O, R = oracle.Oracle(), oracle.RefLib()
    phys, logical = R.cores()
    key = O.sweep(3, 16)
    src = os.path.join(args.dir, "paes_bench_in.bin")
    ct = os.path.join(args.dir, "paes_bench_ct.bin")
    out = os.path.join(args.dir, "paes_bench_out.bin")
    buf = np.empty(args.size, dtype=np.uint8)
    O.counter_fill_into(3, 0, args.size, buf.ctypes.data)
    buf.tofile(src)
    del buf
    res = {"size": args.size, "dir": args.dir, "host_threads": logical}

    def ref_job(inp, outp, direction, workers):
        bi, bo, sec = C.c_uint64(), C.c_uint64(), C.c_double()
        rc = R.L.ref_run_job(inp.encode(), outp.encode(), (C.c_uint8 * 16).from_buffer_copy(key), workers, 1,
                             direction, C.byref(bi), C.byref(bo), C.byref(sec))
        assert rc == 0, rc
        return sec.value

    def ours(inp, outp, direction):
        fn = paes.encrypt_file if direction == 0 else paes.decrypt_file
        return fn(inp, outp, key, workers=1)["seconds"]

    for name, fn in [("reference_threads_enc", lambda: ref_job(src, ct, 0, logical)),
                     ("gpu_enc", lambda: ours(src, ct, 0)),
                     ("reference_threads_dec", lambda: ref_job(ct, out, 1, logical)),
                     ("gpu_dec", lambda: ours(ct, out, 1))]:
        fn()  # warm (page cache, CUDA context, pinned ring)
        samples = [fn() for _ in range(args.reps)]
        kept = R.reject_outliers(samples)
        avg = sum(kept) / len(kept)
        n = args.size if "enc" in name else os.path.getsize(ct)
        res[name] = {"gbs": round(n / avg / 1e9, 3), "mbps": round(n * 8 / avg / 1e6, 1),
                     "seconds": [round(x, 4) for x in samples]}
    # the two strategies must agree byte for byte
    ref_ct = os.path.join(args.dir, "paes_bench_ct_ref.bin")
    ref_job(src, ref_ct, 0, logical)
    paes.encrypt_file(src, ct, key, workers=1)
    res["identical_output"] = open(ref_ct, "rb").read() == open(ct, "rb").read() if args.size <= (4 << 30) else None
    for p in (src, ct, out, ref_ct):
        if os.path.exists(p):
            os.unlink(p)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
