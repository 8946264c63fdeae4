"""Key metrics of every kernel in an `ncu --set full` report, one block per
launch, in the format of profiles/r01_ncu_*.txt; with --traffic also rewrites
profiles/ncu_traffic.json from the first encrypt ecb_kernel launch (the ratio
bench.py scales to its own launch for roofline.traffic).

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep [--traffic] > profiles/rNN_ncu_....txt
"""
import csv
import io
import json
import os
import subprocess
import sys

METRICS = [
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__time_duration.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
    "l1tex__t_requests_pipe_lsu_mem_global_op_st.sum",
    "launch__grid_size",
    "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic",
    "sm__cycles_elapsed.avg.per_second",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True, check=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    head, units = r[0], r[1]
    for row in r[2:]:
        yield {k: (v, u) for k, v, u in zip(head, row, units)}


def main():
    rep = sys.argv[1]
    first_enc = None
    for d in rows(rep):
        name = d["Kernel Name"][0]
        print(f"## {name}")
        for m in METRICS:
            if m in d:
                v, u = d[m]
                print(f"{m:<90} {v} {u}".rstrip())
        print()
        if first_enc is None and "ecb_kernel<0" in name.replace(" ", ""):
            first_enc = d
    if "--traffic" in sys.argv and first_enc is not None:
        def val(m):
            v, u = first_enc[m]
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            return float(v.replace(",", "")) * scale
        n = int(sys.argv[sys.argv.index("--bytes") + 1]) if "--bytes" in sys.argv else (1 << 30)
        dram = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
        alg = 2 * n + 16
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w") as f:
            json.dump({"kernel": "ecb_kernel<enc,2,aligned>", "launch_bytes_plaintext": n,
                       "algorithmic_bytes_per_launch": alg, "dram_bytes_per_launch": dram, "ratio": dram / alg,
                       "source": sys.argv[sys.argv.index("--source") + 1] if "--source" in sys.argv else rep},
                      f, indent=1)
            f.write("\n")


if __name__ == "__main__":
    main()
