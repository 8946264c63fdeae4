"""Generate tests/golden/digests.json -- full-size golden digests for the five
BASELINE.json configs, computed with the REFERENCE's own paes_core
(oracle/_ref/libpaes_ref.so, built from /root/reference/proj/src by
oracle/Makefile).  Inputs come from the oracle's restatement of the
reference's generator (pinned to the survey's digests in tests/test_oracle.py).

    python tests/golden/make_digests.py            # ~3-5 min on 8 cores

Only digests are committed; the GPU tests regenerate inputs on the box and
compare.  Input rules: sweep(seed, n) = first n bytes of
generate_sweep_file(n, seed); key(seed) = sweep(seed, 16).
"""
from __future__ import annotations

import ctypes as C
import hashlib
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "digests.json")
THREADS = os.cpu_count() or 8
O = oracle.Oracle()
R = oracle.RefLib()


def ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def ref_ecb_par(direction: int, src: np.ndarray, dst: np.ndarray, key: bytes) -> None:
    """Reference aes::encrypt_ecb over disjoint slices on THREADS threads."""
    n = src.nbytes
    assert n % 16 == 0
    blocks = n // 16
    parts = []
    off = 0
    for t in range(THREADS):
        share = blocks // THREADS + (1 if t < blocks % THREADS else 0)
        parts.append((off * 16, share * 16))
        off += share
    k = (C.c_uint8 * 16).from_buffer_copy(key)

    def run(p):
        o, ln = p
        if ln:
            rc = R.L.ref_ecb(direction, C.c_void_p(ptr(src) + o), C.c_void_p(ptr(dst) + o), ln, k)
            assert rc == 0

    with ThreadPoolExecutor(THREADS) as ex:
        list(ex.map(run, parts))


def ref_encrypt_chunk_final(pt: np.ndarray, key: bytes) -> np.ndarray:
    """encrypt_chunk(pt, true, ks) == ECB(pt || pad): reference ECB on whole
    blocks in parallel + the reference's own chunk call on the final block."""
    n = pt.nbytes
    nfull = n // 16
    out = np.empty((nfull + 1) * 16, dtype=np.uint8)
    if nfull:
        ref_ecb_par(0, pt[: nfull * 16], out[: nfull * 16], key)
    tail = bytes(pt[nfull * 16:])
    last = R.chunk(0, tail, True, key)
    assert isinstance(last, bytes) and len(last) == 16
    out[nfull * 16:] = np.frombuffer(last, dtype=np.uint8)
    return out


def sha(a) -> str:
    return hashlib.sha256(memoryview(a)).hexdigest()


def sweep_np(seed: int, n: int) -> np.ndarray:
    a = np.empty(max(n, 1), dtype=np.uint8)
    O.sweep_into(seed, n, ptr(a))
    return a[:n]


def main() -> None:
    g: dict = {"generator": "tests/golden/make_digests.py (reference paes_core via oracle/_ref)", "threads": THREADS}
    t0 = time.time()

    # config 1: 64 MiB, seed 0 (cross-checks SURVEY.md A.5)
    pt = sweep_np(0, 64 << 20)
    key = O.sweep(0, 16)
    ct = ref_encrypt_chunk_final(pt, key)
    g["cfg1"] = {"seed": 0, "len": pt.nbytes, "key": key.hex(), "pt_sha256": sha(pt), "ct_sha256": sha(ct),
                 "ct_len": ct.nbytes, "raw_ecb_sha256": None}
    raw = np.empty_like(pt)
    ref_ecb_par(0, pt, raw, key)
    g["cfg1"]["raw_ecb_sha256"] = sha(raw)
    print("cfg1", time.time() - t0, flush=True)

    # config 2: 1 GiB ciphertext of sweep(1, 2^30 - 16)
    pt = sweep_np(1, (1 << 30) - 16)
    key = O.sweep(1, 16)
    ct = ref_encrypt_chunk_final(pt, key)
    assert ct.nbytes == 1 << 30
    g["cfg2"] = {"seed": 1, "pt_len": pt.nbytes, "key": key.hex(), "pt_sha256": sha(pt), "ct_sha256": sha(ct)}
    del pt, ct
    print("cfg2", time.time() - t0, flush=True)

    # config 3: size sweep + 7-byte tail, seed 2
    key = O.sweep(2, 16)
    g["cfg3"] = {"seed": 2, "key": key.hex(), "sizes": []}
    for S in [1 << 10, 64 << 10, 1 << 20, 16 << 20, 256 << 20, 4 << 30]:
        pt = sweep_np(2, S + 7)
        ct = ref_encrypt_chunk_final(pt, key)
        g["cfg3"]["sizes"].append({"S": S, "len": S + 7, "pt_sha256": sha(pt), "ct_sha256": sha(ct),
                                   "ct_len": ct.nbytes, "ct_last16": bytes(ct[-16:]).hex()})
        del pt, ct
        print("cfg3", S, time.time() - t0, flush=True)

    # config 5: 4096 messages, per-message keys
    n = 4096
    lens = O.batch_lengths(4, n)
    hp, hc = hashlib.sha256(), hashlib.sha256()
    per = []
    for i in range(n):
        seed = (4 << 32) + i
        m = sweep_np(seed, lens[i])
        k = O.sweep(seed, 16)
        ct = R.chunk(0, bytes(m), True, k)
        hp.update(memoryview(m))
        hc.update(ct)
        per.append(hashlib.sha256(ct).hexdigest()[:16])
    g["cfg5"] = {"seed": 4, "n": n, "total_len": int(sum(lens)), "lens_sha256": hashlib.sha256(
        np.array(lens, dtype=np.uint64).tobytes()).hexdigest(), "pt_concat_sha256": hp.hexdigest(),
        "ct_concat_sha256": hc.hexdigest(), "ct_msg_sha256_16": per}
    print("cfg5", time.time() - t0, flush=True)

    # config 4: 64 GiB counter stream, seed 3 -- position-keyed checksums of the
    # whole plaintext / padded ciphertext + sha256 of sampled 1 MiB windows.
    total = 64 << 30
    key = O.sweep(3, 16)
    W = 256 << 20
    rng = np.random.default_rng(3)
    win = 1 << 20
    windows = sorted(set([0, total - win] + [int(x) * win for x in rng.integers(0, total // win, 14)]))
    wdig = {}
    cs_pt = cs_ct = 0
    ptb = np.empty(W, dtype=np.uint8)
    ctb = np.empty(W, dtype=np.uint8)
    for off in range(0, total, W):
        O.counter_fill_into(3, off, W, ptr(ptb))
        cs_pt = (cs_pt + O.checksum_ptr(ptr(ptb), W, off // 8)) % (1 << 64)
        ref_ecb_par(0, ptb, ctb, key)
        cs_ct = (cs_ct + O.checksum_ptr(ptr(ctb), W, off // 8)) % (1 << 64)
        for w in windows:
            if off <= w < off + W:
                wdig[str(w)] = sha(ctb[w - off: w - off + win])
        if (off // W) % 32 == 0:
            print("cfg4", off >> 30, "GiB", time.time() - t0, flush=True)
    pad = R.chunk(0, b"", True, key)  # E(16 x 0x10): 64 GiB is block-aligned
    cs_ct = (cs_ct + O.checksum(pad, total // 8)) % (1 << 64)
    g["cfg4"] = {"seed": 3, "len": total, "key": key.hex(), "pt_checksum": cs_pt, "ct_checksum": cs_ct,
                 "pad_block": pad.hex(), "window": win, "window_sha256": wdig}
    print("cfg4 done", time.time() - t0, flush=True)

    with open(OUT, "w") as f:
        json.dump(g, f, indent=1, sort_keys=True)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
