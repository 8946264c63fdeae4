#!/bin/bash
# One GPU call: GPU tests, smoke, the default bench and the reference arm,
# then at most ONE ncu pass, chosen by NCU (one ncu per gpurun call):
#   NCU=launches (default)  launch list of exactly `python bench.py`
#   NCU=full                `ncu --set full` of one encrypt/decrypt/batch launch each
#   NCU=none                no profiler
# Every ncu pass runs only after the same command exited 0 without ncu.
mkdir -p gpurun_out
python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest_gpu rc=$?"; tail -2 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; bench_rc=$?; echo "bench rc=$bench_rc"; tail -c 600 gpurun_out/bench.json
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "bench_ref rc=$?"; tail -c 400 gpurun_out/bench_ref.json
case "${NCU:-launches}" in
  launches)
    if [ $bench_rc -eq 0 ]; then
      ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv \
        python bench.py > gpurun_out/ncu_launch.log 2>&1; echo "ncu_launch rc=$?"
    fi ;;
  full)
    python scripts/profile_kernels.py > gpurun_out/profile_kernels.log 2>&1 && \
      ncu --set full --clock-control none --import-source on -k regex:"ecb_kernel|batch_kernel" -s 3 -c 3 \
        -o gpurun_out/prof_kernels python scripts/profile_kernels.py > gpurun_out/ncu_full.log 2>&1; echo "ncu_full rc=$?" ;;
  none) ;;
esac
