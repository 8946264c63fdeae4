"""Summary of an `ncu --metrics gpu__time_duration.sum --clock-control none --csv`
launch list of `python bench.py` (scripts/gpu_round.sh, NCU=launches) next to
the bench line of the same command run just before it: launches, median and
total time per kernel, and the dominant kernel's share of the step.

    python scripts/launch_summary.py gpurun_out/launches_bench.csv gpurun_out/bench.json "note" > profiles/rNN_launches_..._summary.txt

ncu times are cold-cache and serialised, so only shares are compared with the
bench's own CUDA-event times.
"""
import collections
import csv
import json
import statistics
import sys


def main():
    launches, bench = sys.argv[1], sys.argv[2]
    note = sys.argv[3] if len(sys.argv) > 3 else ""
    with open(launches) as f:
        lines = [ln for ln in f if not ln.startswith("==")]
    groups = collections.OrderedDict()
    for row in csv.DictReader(lines):
        if row.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(row["Metric Value"].replace(",", ""))
        u = row["Metric Unit"]
        ms = v / 1e6 if u in ("ns", "nsecond") else v / 1e3 if u in ("us", "usecond") else v if u in ("ms", "msecond") else v * 1e3
        k = row["Kernel Name"]
        if "ecb_kernel" in k:  # one kernel, three uses: tell them apart by duration
            k += " [64 GiB launch]" if ms > 50 else " [e2e ring piece]" if ms > 0.1 else " [short]"
        groups.setdefault(k, []).append(ms)
    b = json.loads(open(bench).read().strip().splitlines()[-1])
    out = ["ncu --metrics gpu__time_duration.sum --clock-control none -c 400 of `python bench.py`" + (f" ({note})" if note else "") + ";",
           "first 400 kernel launches, cold-cache and serialised by ncu (per-launch times are not bench values)",
           "%-86s %8s %10s %10s" % ("kernel", "launches", "median ms", "total ms")]
    for k, v in groups.items():
        out.append("%-86s %8d %10.3f %10.1f" % (k[:86], len(v), statistics.median(v), sum(v)))
    enc = [v for k, v in groups.items() if "ecb_kernel<0" in k and "64 GiB" in k]
    if enc:
        m = statistics.median(enc[0])
        out += ["", "config-4 encrypt step = one launch: ncu median %.3f ms -> %.1f GB/s;" % (m, 68719476736 / m / 1e6),
                "bench.py (same code, run just before in the same gpurun call): CUDA-event average %.4f ms per launch, "
                "ms_per_step %.4f -> %.2f GB/s; the kernel is 100%% of the step"
                % (b["roofline"]["avg_launch_ms"], b["ms_per_step"], b["value"])]
    print("\n".join(out))


if __name__ == "__main__":
    main()
