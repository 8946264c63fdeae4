"""Generate tests/golden/golden.json from the reference's OWN Python module.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It compiles the reference's pybind11 module ``_paes`` from its sources
(proj/python/paes_module.cpp + proj/src/*.cpp, with ``-include algorithm`` for
the missing include at aes.cpp:248-263) into a scratch dir under /tmp, imports
it, and records input/output vectors.  Only the vectors are committed; the
reference never travels to the GPU box.  Inputs are derived from a fixed
seed so the file is reproducible.
"""
from __future__ import annotations

import hashlib
import importlib
import json
import os
import random
import subprocess
import sys
import sysconfig
import tempfile

REF = "/root/reference/proj"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")


def build_ref_module() -> str:
    import pybind11

    d = tempfile.mkdtemp(prefix="paes_ref_py_")
    ext = sysconfig.get_config_var("EXT_SUFFIX")
    srcs = [f"{REF}/python/paes_module.cpp"] + [f"{REF}/src/{s}.cpp" for s in ("aes", "chunk", "exec", "bench", "report")]
    cmd = ["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-include", "algorithm", f"-I{REF}/include",
           f"-I{pybind11.get_include()}", f"-I{sysconfig.get_paths()['include']}", "-o", f"{d}/_paes{ext}"] + srcs
    subprocess.run(cmd, check=True)
    return d


def main() -> None:
    d = build_ref_module()
    sys.path.insert(0, d)
    _paes = importlib.import_module("_paes")
    rnd = random.Random(20261020)

    def rb(n: int) -> bytes:
        return bytes(rnd.getrandbits(8) for _ in range(n))

    g: dict = {"generator": "tests/golden/make_golden.py (reference _paes built from proj/python/paes_module.cpp)"}

    # FIPS-197 / reference KATs (test_aes.cpp:255-292, test_smoke.py:14-18)
    kats = []
    for key, pt in [("2b7e151628aed2a6abf7158809cf4f3c", "3243f6a8885a308d313198a2e0370734"),
                    ("000102030405060708090a0b0c0d0e0f", "00112233445566778899aabbccddeeff"),
                    ("00" * 16, "00" * 16)]:
        k, p = bytes.fromhex(key), bytes.fromhex(pt)
        kats.append({"key": key, "pt": pt, "ct": _paes.encrypt_block(p, k).hex(),
                     "dec_of_pt": _paes.decrypt_block(p, k).hex()})
    g["block_kats"] = kats

    # key schedules (expand_key) for a few keys
    g["key_schedules"] = []
    for key in ["00" * 16, "2b7e151628aed2a6abf7158809cf4f3c"] + [rb(16).hex() for _ in range(6)]:
        g["key_schedules"].append({"key": key, "rk": "".join(r.hex() for r in _paes.expand_key(bytes.fromhex(key)))})

    # encrypt_bytes (always-pad) across ragged lengths, with decrypt round trips
    g["bytes"] = []
    for n in list(range(0, 49)) + [63, 64, 65, 255, 256, 257, 1000, 1031, 4096, 65543]:
        key, data = rb(16), rb(n)
        ct = _paes.encrypt_bytes(data, key)
        assert _paes.decrypt_bytes(ct, key) == data
        entry = {"key": key.hex(), "len": n}
        entry["pt"] = data.hex()  # <= 64 KiB, embedded
        if n <= 300:
            entry["ct"] = ct.hex()
        else:
            entry["ct_sha256"] = hashlib.sha256(ct).hexdigest()
        g["bytes"].append(entry)

    # wrong-key decrypt -> ValueError (PaddingError) (test_smoke.py:28-31)
    wrong = []
    for i in range(8):
        key, data = rb(16), rb(11 + 7 * i)
        ct = _paes.encrypt_bytes(data, key)
        bad = bytes([key[0] ^ 0xFF]) + key[1:]
        try:
            _paes.decrypt_bytes(ct, bad)
            outcome = "ok"
        except ValueError:
            outcome = "PaddingError"
        wrong.append({"key": key.hex(), "bad_key": bad.hex(), "ct": ct.hex(), "outcome": outcome})
    g["wrong_key"] = wrong

    # pad / unpad edge cases (test_chunk.cpp:128-163)
    pads = []
    for n in range(0, 40):
        data = rb(n)
        pads.append({"in": data.hex(), "out": _paes.pkcs7_pad(data).hex()})
    g["pad"] = pads
    unpads = []
    for case in ["", "01" * 15, "00" * 16, "11" * 16, "04" * 13 + "05" + "04" * 2, "10" * 16, "aa" * 15 + "01",
                 "bb" * 12 + "04" * 4, "cc" * 16 + "02" * 16]:
        try:
            out = _paes.pkcs7_unpad(bytes.fromhex(case)).hex()
            res = {"ok": True, "out": out}
        except ValueError:
            res = {"ok": False}
        unpads.append({"in": case, **res})
    g["unpad"] = unpads

    # plan_chunks (test_chunk.cpp:57-117 examples + a sampled dense grid)
    plans = []
    for total, w in [(1024, 4), (1000, 4), (16, 1), (0, 1), (0, 2), (0, 33), (16, 33), (17, 33), (1024, 65),
                     (1 << 26, 8), ((1 << 30) - 16, 8), (64 << 30, 8), (64 << 30, 3)] + \
                    [(rnd.randrange(0, 1025), rnd.randrange(1, 34)) for _ in range(200)]:
        plans.append({"total": total, "workers": w,
                      "chunks": [[c["offset"], c["raw_len"], c["padded_len"], bool(c["is_final"])]
                                 for c in _paes.plan_chunks(total, w)]})
    g["plans"] = plans

    # reject_outliers (bench.cpp:49-79; test_smoke.py:48-51)
    ro = []
    for s in [[10, 10, 10, 10], [9, 10, 11, 12, 30], [10, 10, 10, 100], [1.0, 2.0, 3.0], [5.0],
              [1.0, 1.0, 1.0, 50.0, 60.0, 70.0]] + [[round(rnd.uniform(0.5, 2.0), 4) for _ in range(rnd.randrange(3, 12))]
                                                    for _ in range(20)]:
        ro.append({"in": s, "out": _paes.reject_outliers(s)})
    g["reject_outliers"] = ro

    # the bench report's CSV contract (report.hpp:12-13)
    g["csv_header"] = _paes.csv_header()

    with open(OUT, "w") as f:
        json.dump(g, f, indent=0, sort_keys=True)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
