"""CPU checks of bench.py's helpers: the rank shard rule, checksum summation
mod 2^64, NUMA cpulist parsing and binding fallback, clock-sampler device id
and the clock-reason verdict.  No GPU, no compute calls."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_cpulist_parsing():
    assert sorted(bench._cpulist("0-3,8,10-11\n")) == [0, 1, 2, 3, 8, 10, 11]
    assert bench._cpulist("") == set()
    assert sorted(bench._cpulist("5")) == [5]


def test_numa_binding_never_raises_without_a_gpu():
    import torch

    before = os.sched_getaffinity(0)
    msg = bench.bind_to_gpu_numa(torch, 0)
    assert msg.startswith("unbound") or msg.startswith("node")
    if msg.startswith("unbound"):
        assert os.sched_getaffinity(0) == before


def test_clock_sampler_falls_back_to_the_ordinal_without_cuda():
    s = bench.ClockSampler(3)
    assert s.device == "3" or ":" in s.device


def test_rank_shards_cover_the_stream(paes):
    total = 64 << 30
    for world in (1, 2, 4, 8):
        shards = [bench.rank_shard(total, world, r, paes.plan_chunks) for r in range(world)]
        assert sum(s["raw_len"] for s in shards) == total
        assert [s["is_final"] for s in shards] == [False] * (world - 1) + [True]
        assert all(s["offset"] % 16 == 0 for s in shards)
    assert bench.rank_shard(16, 4, 3, paes.plan_chunks)["raw_len"] == 0  # more ranks than blocks


def test_checksum_sum_wraps_mod_2_64():
    class One:
        def reduce(self, v, op):
            return v

    for cs in (0, 1, (1 << 63) - 1, 1 << 63, (1 << 64) - 1):
        assert bench.sum_checksums(One(), cs) == cs


def test_clock_verdict():
    ok = {"sm_mhz": 1965.0, "sm_max_mhz": 1965.0, "reasons": []}
    assert not bench.clocks_suspect(ok)
    assert not bench.clocks_suspect({**ok, "reasons": ["sw_power_cap"], "sm_mhz": 1400.0})  # kept, noted
    for r in ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"):
        assert bench.clocks_suspect({**ok, "reasons": [r]})
    assert bench.clocks_suspect({**ok, "sm_mhz": 1100.0})  # pinned low, no reason
    assert not bench.clocks_suspect({"sm_mhz": None, "sm_max_mhz": 1965.0, "reasons": ["nvidia-smi unavailable"]})


def test_clock_sampler_summary_parses_nvidia_smi_rows():
    import tempfile

    s = bench.ClockSampler(0)
    s.proc = object()
    s.out = tempfile.TemporaryFile(mode="w+")
    rows = ["0, 1965, 1965, 700.5, 0x0, Not Active, Not Active, Not Active, Not Active",
            "0, 1965, 1965, 710.0, 0x0, Not Active, Not Active, Not Active, Active",
            "0, 600, 1965, 90.0, 0x0, Not Active, Not Active, Not Active, Not Active",  # idle sample
            "garbage"]
    s.out.write("\n".join(rows) + "\n")
    d = s.summary(1965.0)
    assert d["samples"] == 3 and d["samples_under_load"] == 2
    assert d["sm_mhz"] == 1965.0 and d["sm_max_mhz"] == 1965.0 and d["power_w_max"] == 710.0
    assert d["reasons"] == ["sw_power_cap"]
