"""GPU cells in the reference's bench/report harness.

Restates the measurement contract of the reference's harness so GPU and CPU
results sit in one report: the same CSV header and column formats
(report.hpp:12-13, report.cpp:35-45), the same repeat / reject_outliers /
mean method and throughput formulas (bench.cpp:81-107), and a Table-I style
summary (report.cpp:74-129, simplified).  The SVG charts are out of scope.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Iterable, List

from .paes import reject_outliers

CSV_HEADER = "file_size_bytes,workers,strategy,reps,retained,avg_seconds,throughput_mbps,throughput_per_core_mbps"


@dataclass
class BenchRecord:
    """bench.hpp:37-48."""

    file_size: int
    workers: int
    strategy: str
    samples: List[float] = field(default_factory=list)
    retained: List[float] = field(default_factory=list)
    avg_seconds: float = 0.0
    throughput_mbps: float = 0.0
    throughput_per_core_mbps: float = 0.0
    failed: bool = False
    error: str = ""


def measure_cell(run: Callable[[], float], file_size: int, workers: int, strategy: str, reps: int,
                 cores: int) -> BenchRecord:
    """measure_cell (bench.cpp:81-107): `run` returns one job's wall seconds."""
    if reps < 3:
        raise ValueError("measure_cell: repetitions must be >= 3")
    if cores <= 0:
        raise ValueError("measure_cell: core count must be >= 1")
    rec = BenchRecord(file_size, workers, strategy)
    try:
        rec.samples = [float(run()) for _ in range(reps)]
    except Exception as e:  # a failed cell is recorded, never aborts the sweep
        rec.failed, rec.error = True, str(e)
        return rec
    rec.retained = reject_outliers(rec.samples)
    rec.avg_seconds = sum(rec.retained) / len(rec.retained)
    rec.throughput_mbps = file_size * 8.0 / (rec.avg_seconds * 1e6)
    rec.throughput_per_core_mbps = rec.throughput_mbps / cores
    return rec


def to_csv(records: Iterable[BenchRecord]) -> str:
    """report.cpp:35-45: successful records, seconds %.6f, throughput %.1f."""
    lines = [CSV_HEADER]
    for r in records:
        if r.failed:
            continue
        lines.append(f"{r.file_size},{r.workers},{r.strategy},{len(r.samples)},{len(r.retained)},"
                     f"{r.avg_seconds:.6f},{r.throughput_mbps:.1f},{r.throughput_per_core_mbps:.1f}")
    return "\n".join(lines) + "\n"


def parse_csv(text: str) -> List[BenchRecord]:
    """report.cpp:47-72 (reps/retained come back as counts)."""
    lines = text.splitlines()
    if not lines or lines[0] != CSV_HEADER:
        raise ValueError("parse_csv: bad header")
    out = []
    for line in lines[1:]:
        if not line:
            continue
        f = line.split(",")
        if len(f) != 8:
            raise ValueError("parse_csv: bad row: " + line)
        r = BenchRecord(int(f[0]), int(f[1]), f[2], samples=[0.0] * int(f[3]), retained=[0.0] * int(f[4]),
                        avg_seconds=float(f[5]), throughput_mbps=float(f[6]), throughput_per_core_mbps=float(f[7]))
        out.append(r)
    return out


def summary_table(records: Iterable[BenchRecord], cores: int) -> str:
    """Best throughput per strategy (Mb/s and per core), Table-I style."""
    records = list(records)
    best = {}
    for r in records:
        if r.failed:
            continue
        if r.strategy not in best or r.throughput_mbps > best[r.strategy].throughput_mbps:
            best[r.strategy] = r
    rows = [f"Results ({cores} logical cores)", "strategy      best Mb/s   per-core Mb/s   workers   file size"]
    for s, r in sorted(best.items()):
        rows.append(f"{s:<12} {r.throughput_mbps:>10.1f} {r.throughput_per_core_mbps:>15.1f} {r.workers:>9} "
                    f"{r.file_size:>11}")
    failed = [r for r in records if r.failed]
    for r in failed:
        rows.append(f"FAILED {r.strategy} workers={r.workers} size={r.file_size}: {r.error}")
    return "\n".join(rows) + "\n"
