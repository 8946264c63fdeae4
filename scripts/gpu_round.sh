#!/bin/bash
# One GPU call: full GPU tests, smoke, default bench, reference arm, then the
# ncu launch list of the bench and one full capture of the encrypt kernel.
mkdir -p gpurun_out
python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest_gpu rc=$?"; tail -2 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -c 600 gpurun_out/bench.log
python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "bench_ref rc=$?"; tail -c 400 gpurun_out/bench_ref.log
if [ "${NCU:-1}" = "1" ]; then
  ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches.csv python bench.py --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo "ncu_launch rc=$?"
  python bench.py --total-bytes 1073741824 --steps 3 --warmup 3 --no-e2e --no-cpu --no-decrypt > gpurun_out/bench1g.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:ecb_kernel -s 2 -c 1 -o gpurun_out/prof_enc python bench.py --total-bytes 1073741824 --steps 3 --warmup 3 --no-e2e --no-cpu --no-decrypt > gpurun_out/ncu_full.log 2>&1; echo "ncu_full rc=$?"
fi
