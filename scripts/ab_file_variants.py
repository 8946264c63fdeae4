"""A/B of run_job builds on the same input file: alternates library variants
(python scripts/ab_file_variants.py LIB_A LIB_B ... --size N --reps R), one
subprocess per run so each loads its own libpaes_cuda.so; the second of two
jobs per process is timed.  Prints one JSON
line of per-variant job seconds (JobOutcome.seconds, exec.cpp:144-200)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

ONE = r'''
import os, sys, json
sys.path.insert(0, %(root)r)
from paper_1403_7295_b200 import _native as N
N.lib_path = lambda: %(lib)r
from paper_1403_7295_b200 import paes
paes.encrypt_file(%(inp)r, %(out)r, bytes(range(16)), workers=1)  # warm: context, rings, pinned slots
os.unlink(%(out)r)
o = paes.encrypt_file(%(inp)r, %(out)r, bytes(range(16)), workers=1)
print(json.dumps(o))
'''


def main():
    args = sys.argv[1:]
    size, reps, libs = 4 << 30, 4, []
    i = 0
    while i < len(args):
        if args[i] == "--size":
            size = int(args[i + 1]); i += 2
        elif args[i] == "--reps":
            reps = int(args[i + 1]); i += 2
        else:
            libs.append(os.path.abspath(args[i])); i += 1
    inp, out = "/dev/shm/paes_ab_in", "/dev/shm/paes_ab_out"
    with open(inp, "wb") as f:
        chunk = os.urandom(64 << 20)
        for _ in range(size // len(chunk)):
            f.write(chunk)
    res = {lib: [] for lib in libs}
    for _ in range(reps):
        for lib in libs:
            r = subprocess.run([sys.executable, "-c", ONE % dict(root=ROOT, lib=lib, inp=inp, out=out)],
                               capture_output=True, text=True, check=True)
            res[lib].append(round(json.loads(r.stdout.strip().splitlines()[-1])["seconds"], 4))
            os.unlink(out)
    os.unlink(inp)
    print(json.dumps({"size": size, "seconds": {os.path.relpath(k, ROOT): v for k, v in res.items()},
                      "gbs_best": {os.path.relpath(k, ROOT): round(size / min(v) / 1e9, 2) for k, v in res.items()}}))


if __name__ == "__main__":
    main()
