"""The reference's `paes bench` sweep (bench.cpp:127-178) with a GPU cell:
sizes x workers x strategies, file -> file run_job per repetition, reported
in the reference's CSV format so CPU and GPU sit in one report.

    python scripts/bench_sweep.py [--sizes 64M,1G] [--reps 5] [--dir /dev/shm] [--out profiles/r01_sweep]

strategy "threads" = the reference's own run_job(Threaded, W) (oracle/_ref),
strategy "gpu" = paes_cuda_run_job on the visible B200s.  Inputs are the
reference's sweep files (generate_sweep_file, default seed
0x7061657300000001, bench.hpp:28).
"""
from __future__ import annotations

import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_1403_7295_b200 import paes, report  # noqa: E402

SEED = 0x7061657300000001


def parse_size(s: str) -> int:
    mult = {"K": 1 << 10, "M": 1 << 20, "G": 1 << 30}
    return int(s[:-1]) * mult[s[-1]] if s[-1] in mult else int(s)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="64M,1G")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--dir", default="/dev/shm")
    ap.add_argument("--out", default="gpurun_out/sweep")
    args = ap.parse_args()
    R = oracle.RefLib()
    _, logical = R.cores()
    key = bytes(16)  # BenchConfig.key default (bench.hpp:24)
    workers_cpu = sorted({1, max(1, logical // 4), logical})
    records = []
    for size in [parse_size(s) for s in args.sizes.split(",")]:
        path = os.path.join(args.dir, f"sweep_{size}.bin")
        buf = np.empty(size, dtype=np.uint8)
        paes.sweep_into(SEED, size, buf.ctypes.data)
        buf.tofile(path)
        del buf
        out = os.path.join(args.dir, "bench_out.tmp")

        def ref_run(w):
            bi, bo, sec = C.c_uint64(), C.c_uint64(), C.c_double()
            rc = R.L.ref_run_job(path.encode(), out.encode(), (C.c_uint8 * 16).from_buffer_copy(key), w, 1, 0,
                                 C.byref(bi), C.byref(bo), C.byref(sec))
            if rc:
                raise RuntimeError(f"reference run_job rc={rc}")
            return sec.value

        for w in workers_cpu:
            records.append(report.measure_cell(lambda: ref_run(w), size, w, "threads", args.reps, logical))
        ngpu = paes.device_count()
        paes.encrypt_file(path, out, key, workers=ngpu, strategy="gpu")  # warm-up (context, pinned ring)
        records.append(report.measure_cell(lambda: paes.encrypt_file(path, out, key, workers=ngpu,
                                                                     strategy="gpu")["seconds"],
                                           size, ngpu, "gpu", args.reps, logical))
        for p in (path, out):
            if os.path.exists(p):
                os.unlink(p)
    os.makedirs(args.out, exist_ok=True)
    csv = report.to_csv(records)
    assert [(r.strategy, r.workers) for r in report.parse_csv(csv)] == \
        [(r.strategy, r.workers) for r in records if not r.failed]
    open(os.path.join(args.out, "report.csv"), "w").write(csv)
    open(os.path.join(args.out, "summary.txt"), "w").write(report.summary_table(records, logical))
    print(csv)
    print(report.summary_table(records, logical))


if __name__ == "__main__":
    main()
