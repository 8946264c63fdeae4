"""Configs 1, 2, 3, 5 (+ pageable and file -> file legs) on one B200, without
the 64 GiB headline: the same code bench.py runs for its "configs" object
(bench.ConfigBench), for iterating on one config.

    python scripts/bench_configs.py [--configs 1,2,3,5,pageable,file] [--steps K] [--warmup W]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1403_7295_b200 import paes  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,5")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    cb = bench.ConfigBench(args, torch, paes, 0, sms)
    fns = {"1": cb.cfg1, "2": cb.cfg2, "3": cb.cfg3, "5": cb.cfg5, "pageable": cb.pageable, "file": cb.file_e2e}
    want = args.configs.split(",")
    if ("pageable" in want or "file" in want) and "3" not in want:
        want = ["3"] + want  # those legs reuse config 3's 4 GiB input
    for c in want:
        with bench.ClockSampler(0) as clk:
            r = fns[c]()
        r["clocks"] = clk.summary(1965.0)
        if r["clocks"].get("sm_mhz"):
            cb.clk_mhz = r["clocks"]["sm_mhz"]
        print(json.dumps({c: r}), flush=True)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
