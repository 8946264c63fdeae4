"""Secondary BASELINE.json configs on one B200 (bench.py measures config 4).

    python scripts/bench_configs.py [--configs 1,2,3,5] [--steps K] [--warmup W]

Prints one JSON line per config with the same keys as bench.py where they
apply (value = device-resident GB/s of input bytes, e2e through the public
host-pointer call, kernel-only GB/s from CUDA events, roofline fraction of
the shared-memory lookup pipe at the sampled SM clock).  Every config first
checks its own output against tests/golden/digests.json (computed by the
reference's paes_core).
"""
from __future__ import annotations

import argparse
import ctypes as C
import hashlib
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1403_7295_b200 import _native as N  # noqa: E402
from paper_1403_7295_b200 import paes  # noqa: E402

GiB, MiB = 1 << 30, 1 << 20
DIG = json.load(open(os.path.join(ROOT, "tests", "golden", "digests.json")))


def pipe_peak(clk_mhz: float) -> float:
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    return sms * clk_mhz * 1e6 * bench.LDS_PER_CLK_PER_SM / bench.LOOKUPS_PER_BLOCK * 16 / 1e9


def timed(fn, steps, warmup, stream):
    """Device-resident timing as bench.py does it: one CUDA event pair around
    `steps` calls queued back to back on `stream`.  Returns the per-step
    device time (ms, as a list so callers can average), the host wall time of
    the loop (API-level throughput, including Python call overhead and any
    per-call sync such as a final decrypt's trailer check) and the clocks."""
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with bench.ClockSampler(0) as clk:
        t = time.perf_counter()
        a.record(stream)
        for _ in range(steps):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t
    per = a.elapsed_time(b) / steps
    return [per] * steps, wall, clk.summary(1965.0)


def host_e2e(direction, host_ptr, n, final, rk, steps, out_ptr=None):
    """In place for encrypt (repeated encryption is the same work); decrypt
    needs a separate output so every step sees valid ciphertext."""
    L = N.load()
    olen = C.c_uint64()
    out_ptr = out_ptr or host_ptr

    def call():
        rc = L.paes_cuda_chunk(direction, host_ptr, n, int(final), rk, out_ptr, C.byref(olen), 1)
        if rc:
            raise RuntimeError(N.last_error())

    call()
    t = time.perf_counter()
    for _ in range(steps):
        call()
    el = time.perf_counter() - t
    return n * steps / el / 1e9, olen.value


def line(cfg, workload, value, ms, wall, clk, steps, warmup, n_in, e2e, extra):
    kern_gbs = n_in / (statistics.mean(ms) / 1e3) / 1e9
    clk_mhz = clk.get("sm_mhz") or 1965.0
    out = {"metric": f"AES-128 ECB {cfg} throughput", "config": {"workload": workload}, "value": round(value, 2),
           "unit": "GB/s", "n_gpus": 1, "steps": steps, "warmup": warmup,
           "ms_per_step": round(statistics.mean(ms), 4), "kernel_gbs": round(kern_gbs, 2),
           "api_wall_gbs": round(n_in * steps / wall / 1e9, 2),
           "pipe_frac": round(kern_gbs / pipe_peak(clk_mhz), 4), "clocks": clk, "e2e": e2e}
    out.update(extra)
    return out


def cfg1(args, s):
    d = DIG["cfg1"]
    n = d["len"]
    key = paes.sweep(0, 16)
    rk = paes.round_keys(key)
    host = torch.empty(n + 32, dtype=torch.uint8, pin_memory=True)
    paes.sweep_into(0, n, host.data_ptr())
    src = host[:n].cuda()
    ct = torch.empty(n + 16, dtype=torch.uint8, device="cuda")
    back = torch.empty(n + 16, dtype=torch.uint8, device="cuda")
    assert paes.chunk_device(0, src.data_ptr(), n, True, rk, ct.data_ptr()) == n + 16
    ok = hashlib.sha256(ct.cpu().numpy().tobytes()).hexdigest() == d["ct_sha256"]
    ms, wall, clk = timed(lambda: paes.chunk_device(0, src.data_ptr(), n, True, rk, ct.data_ptr(), 0, s.cuda_stream),
                          args.steps, args.warmup, s)
    msd, walld, _ = timed(lambda: paes.chunk_device(1, ct.data_ptr(), n + 16, True, rk, back.data_ptr(), 0,
                                                      s.cuda_stream), args.steps, args.warmup, s)
    assert paes.count_mismatch_device(back.data_ptr(), src.data_ptr(), n) == 0
    e2e, _ = host_e2e(0, host.data_ptr(), n, True, rk, args.steps)
    return line("encrypt (config 1, 64 MiB) + decrypt round trip", "config1: sweep(0, 64 MiB), key sweep(0,16)",
                n * args.steps / (sum(ms) / 1e3) / 1e9, ms, wall, clk, args.steps, args.warmup, n,
                {"value": round(e2e, 2), "unit": "GB/s", "h2d_bytes_per_step": n, "d2h_bytes_per_step": n + 16},
                {"parity": "ok" if ok else "MISMATCH", "decrypt_value": round((n + 16) * args.steps / (sum(msd) / 1e3) / 1e9, 2),
                 "decrypt_kernel_gbs": round((n + 16) / (statistics.mean(msd) / 1e3) / 1e9, 2)})


def cfg2(args, s):
    d = DIG["cfg2"]
    n = d["pt_len"]
    key = paes.sweep(1, 16)
    rk = paes.round_keys(key)
    pt = np.empty(n, dtype=np.uint8)
    paes.sweep_into(1, n, pt.ctypes.data)
    src = torch.from_numpy(pt).cuda()
    ct = torch.empty(GiB, dtype=torch.uint8, device="cuda")
    out = torch.empty(GiB, dtype=torch.uint8, device="cuda")
    paes.chunk_device(0, src.data_ptr(), n, True, rk, ct.data_ptr())
    ok = hashlib.sha256(ct.cpu().numpy().tobytes()).hexdigest() == d["ct_sha256"]
    # device-resident final decrypt (includes the trailer check + its 4-byte readback each step)
    ms, wall, clk = timed(lambda: paes.chunk_device(1, ct.data_ptr(), GiB, True, rk, out.data_ptr(), 0,
                                                    s.cuda_stream), args.steps, args.warmup, s)
    assert paes.count_mismatch_device(out.data_ptr(), src.data_ptr(), n - n % 16) == 0
    host = torch.empty(GiB + 32, dtype=torch.uint8, pin_memory=True)
    host[:GiB].copy_(ct)
    hout = torch.empty(GiB + 32, dtype=torch.uint8, pin_memory=True)
    e2e, olen = host_e2e(1, host.data_ptr(), GiB, True, rk, args.steps, hout.data_ptr())
    assert olen == n
    return line("decrypt (config 2, 1 GiB ciphertext)", "config2: decrypt of the reference's 1 GiB ciphertext of "
                "sweep(1, 1 GiB-16)", GiB * args.steps / (sum(ms) / 1e3) / 1e9, ms, wall, clk, args.steps, args.warmup, GiB,
                {"value": round(e2e, 2), "unit": "GB/s", "h2d_bytes_per_step": GiB, "d2h_bytes_per_step": GiB},
                {"parity": "ok" if ok else "MISMATCH"})


def cfg3(args, s):
    d = {e["S"]: e for e in DIG["cfg3"]["sizes"]}
    key = paes.sweep(2, 16)
    rk = paes.round_keys(key)
    rows = []
    for S in sorted(d):
        n = S + 7
        host = torch.empty(n + 48, dtype=torch.uint8, pin_memory=True)
        paes.sweep_into(2, n, host.data_ptr())
        src = host[:n].cuda()
        m = (n // 16 + 1) * 16
        ct = torch.empty(m, dtype=torch.uint8, device="cuda")
        assert paes.chunk_device(0, src.data_ptr(), n, True, rk, ct.data_ptr()) == m
        ok = hashlib.sha256(ct.cpu().numpy().tobytes()).hexdigest() == d[S]["ct_sha256"]
        steps = args.steps if S >= 16 * MiB else max(args.steps, 50)
        ms, wall, clk = timed(lambda: paes.chunk_device(0, src.data_ptr(), n, True, rk, ct.data_ptr(), 0,
                                                        s.cuda_stream), steps, args.warmup, s)
        e2e, _ = host_e2e(0, host.data_ptr(), n, True, rk, min(steps, 20) if S >= 16 * MiB else steps)
        rows.append({"size": n, "device_gbs": round(n * steps / (sum(ms) / 1e3) / 1e9, 3), "api_wall_gbs": round(n * steps / wall / 1e9, 3),
                     "kernel_us": round(statistics.mean(ms) * 1e3, 2), "e2e_gbs": round(e2e, 3),
                     "parity": "ok" if ok else "MISMATCH", "sm_mhz": clk.get("sm_mhz")})
        del host, src, ct
        torch.cuda.empty_cache()
    return {"metric": "AES-128 ECB encrypt size sweep (config 3)", "config": {"workload": "config3: sweep(2, S+7), "
            "S = 1 KiB .. 4 GiB, key sweep(2,16), always-pad (nine 0x09)"}, "unit": "GB/s", "rows": rows}


def cfg5(args, s):
    d = DIG["cfg5"]
    n = d["n"]
    lens = paes.batch_lengths(4, n)
    in_off, out_off, oi, oo = [], [], 0, 0
    for L in lens:
        in_off.append(oi)
        out_off.append(oo)
        oi += L
        oo += L + 16
    host = torch.empty(oi + 16, dtype=torch.uint8, pin_memory=True)
    rks = bytearray()
    for i in range(n):
        seed = (4 << 32) + i
        paes.sweep_into(seed, lens[i], host.data_ptr() + in_off[i])
        rks += paes.round_keys(paes.sweep(seed, 16))
    rks = bytes(rks)
    src = host[:oi].cuda()
    dst = torch.empty(oo, dtype=torch.uint8, device="cuda")
    back = torch.empty(oo, dtype=torch.uint8, device="cuda")
    paes.ecb_batch(0, src.data_ptr(), dst.data_ptr(), in_off, out_off, lens, rks, True)
    torch.cuda.synchronize()
    out = dst.cpu().numpy()
    hc = hashlib.sha256()
    for i in range(n):
        hc.update(memoryview(out[out_off[i]:out_off[i] + lens[i] + 16]))
    ok = hc.hexdigest() == d["ct_concat_sha256"]
    # one-shot API (descriptor table + key words built and uploaded every call)
    ms1, wall1, _ = timed(lambda: paes.ecb_batch(0, src.data_ptr(), dst.data_ptr(), in_off, out_off, lens, rks, True,
                                                 0, s.cuda_stream), args.steps, args.warmup, s)
    # prepared plan: one launch per step
    enc_plan = paes.BatchPlan(0, in_off, out_off, lens, rks, True)
    ms, wall, clk = timed(lambda: enc_plan.run(src.data_ptr(), dst.data_ptr(), s.cuda_stream), args.steps,
                          args.warmup, s)
    clen = [L + 16 for L in lens]
    dec_plan = paes.BatchPlan(1, out_off, out_off, clen, rks, True)
    msd, walld, _ = timed(lambda: dec_plan.run(dst.data_ptr(), back.data_ptr(), s.cuda_stream), args.steps,
                          args.warmup, s)
    assert dec_plan.run(dst.data_ptr(), back.data_ptr(), s.cuda_stream) == lens
    # e2e through the public host-pointer batch call: message groups pipelined
    # H2D / fused launch / D2H over the stream ring (paes_cuda_batch_host)
    hout = torch.empty(oo, dtype=torch.uint8, pin_memory=True)
    paes.ecb_batch_host(0, host.data_ptr(), hout.data_ptr(), in_off, out_off, lens, rks, True)
    assert paes.count_mismatch_device(dst.data_ptr(), hout.cuda().data_ptr(), oo) == 0
    t = time.perf_counter()
    for _ in range(args.steps):
        paes.ecb_batch_host(0, host.data_ptr(), hout.data_ptr(), in_off, out_off, lens, rks, True)
    e2e = oi * args.steps / (time.perf_counter() - t) / 1e9
    return line("batch encrypt (config 5, 4096 messages, per-message keys)",
                "config5: 4096 msgs, log-uniform 4 KiB..4 MiB, keys sweep((4<<32)+i,16), one fused launch",
                oi * args.steps / (sum(ms) / 1e3) / 1e9, ms, wall, clk, args.steps, args.warmup, oi,
                {"value": round(e2e, 2), "unit": "GB/s", "h2d_bytes_per_step": oi, "d2h_bytes_per_step": oo,
                 "api": "paes_cuda_batch_host (pinned host; ~64 MiB message groups pipelined over 3 streams)"},
                {"parity": "ok" if ok else "MISMATCH", "total_bytes": oi,
                 "one_shot_api_gbs": round(oi * args.steps / wall1 / 1e9, 2), "one_shot_device_gbs": round(oi * args.steps / (sum(ms1) / 1e3) / 1e9, 2),
                 "one_shot_ms": round(statistics.mean(ms1), 3),
                 "value_is": "prepared plan (paes_cuda_batch_plan_run): one launch per step",
                 "decrypt_value": round(oo * args.steps / (sum(msd) / 1e3) / 1e9, 2),
                 "decrypt_kernel_gbs": round(oo / (statistics.mean(msd) / 1e3) / 1e9, 2)})


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,5")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    s = torch.cuda.Stream()
    fns = {"1": cfg1, "2": cfg2, "3": cfg3, "5": cfg5}
    for c in args.configs.split(","):
        r = fns[c](args, s)
        print(json.dumps(r), flush=True)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
