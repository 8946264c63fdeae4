"""CPU: the report harness restates the reference's CSV contract and the
measure_cell method (test_bench.cpp:48-97 style: an injected fake runner)."""
import pytest

from paper_1403_7295_b200 import report


def test_csv_header_is_the_references(golden):
    assert report.CSV_HEADER == golden["csv_header"]
    from paper_1403_7295_b200 import paes

    assert paes.csv_header() == golden["csv_header"]  # the _paes mirror's entry (paes_module.cpp:151)


def test_measure_cell_with_scripted_samples():
    samples = iter([1.0, 1.0, 1.0, 10.0, 1.0])  # the 10 s outlier is rejected (bench.cpp:49-79)
    rec = report.measure_cell(lambda: next(samples), 1_000_000, 4, "gpu", 5, 8)
    assert rec.retained == [1.0, 1.0, 1.0, 1.0]
    assert rec.avg_seconds == pytest.approx(1.0)
    assert rec.throughput_mbps == pytest.approx(8.0)  # bytes*8 / (s*1e6)
    assert rec.throughput_per_core_mbps == pytest.approx(1.0)
    with pytest.raises(ValueError):
        report.measure_cell(lambda: 1.0, 1, 1, "gpu", 2, 8)


def test_failed_cell_is_recorded_not_raised():
    def boom():
        raise RuntimeError("no device")

    rec = report.measure_cell(boom, 10, 1, "gpu", 3, 8)
    assert rec.failed and "no device" in rec.error
    assert report.to_csv([rec]) == report.CSV_HEADER + "\n"
    assert "FAILED gpu" in report.summary_table([rec], 8)


def test_csv_round_trip_and_formats():
    recs = [report.measure_cell(lambda: 0.5, 1 << 20, w, s, 3, 16) for w, s in [(1, "threads"), (16, "threads"),
                                                                               (1, "gpu")]]
    text = report.to_csv(recs)
    row = text.splitlines()[1].split(",")
    assert row[5] == "0.500000" and row[6] == "16.8"  # %.6f seconds, %.1f Mb/s (report.cpp:35-45)
    back = report.parse_csv(text)
    assert [(r.file_size, r.workers, r.strategy, len(r.samples)) for r in back] == \
        [(1 << 20, 1, "threads", 3), (1 << 20, 16, "threads", 3), (1 << 20, 1, "gpu", 3)]
    with pytest.raises(ValueError):
        report.parse_csv("bad,header\n")
    assert "gpu" in report.summary_table(recs, 16)
