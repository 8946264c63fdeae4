#!/usr/bin/env bash
# ThreadSanitizer run of the host runtime: builds a TSAN-instrumented variant
# of libpaes_cuda.so (tune/tsan/, host code only -- kernels are unchanged) and
# tests/cpp/stress_threads.cpp against it, then (with `run`) executes the
# stress on the GPU.  Writes gpurun_out/tsan_stress.log.
#   bash scripts/tsan_stress.sh build        # here (nvcc, no GPU)
#   bash scripts/tsan_stress.sh run          # on the B200 box
set -euo pipefail
cd "$(dirname "$0")/.."
if [ "${1:-build}" = build ]; then
  python - <<'PY'
import sys; sys.path.insert(0, ".")
from paper_1403_7295_b200 import build
build.build(out_lib="tune/tsan/libpaes_cuda.so", host_flags=["-fsanitize=thread", "-g"])
PY
  /usr/bin/g++ -std=c++17 -O1 -g -fsanitize=thread -Iinclude -I/usr/local/cuda/include tests/cpp/stress_threads.cpp \
    -o tune/tsan/stress_threads -Ltune/tsan -lpaes_cuda -L/usr/local/cuda/lib64 -lcudart \
    -Wl,-rpath,'$ORIGIN' -Wl,-rpath,/usr/local/cuda/lib64
  echo "built tune/tsan/stress_threads"
else
  mkdir -p gpurun_out
  # The CUDA driver's launch path copies kernel parameters into driver-owned
  # buffers under its own synchronisation, which TSAN cannot see; races whose
  # frames are all inside libcuda are suppressed (our frames stay checked).
  printf 'race:libcuda.so\n' > tune/tsan/suppressions.txt
  TSAN_OPTIONS="halt_on_error=0 second_deadlock_stack=1 report_signal_unsafe=0 suppressions=tune/tsan/suppressions.txt print_suppressions=1" \
    ./tune/tsan/stress_threads 8 40 > gpurun_out/tsan_stress.log 2>&1 || true
  echo "tsan warnings: $(grep -c 'WARNING: ThreadSanitizer' gpurun_out/tsan_stress.log || true)"
  grep -E "^stress:|Suppression|matched" gpurun_out/tsan_stress.log | head -5 || true
fi
