#!/usr/bin/env bash
# Sanitizer runs of the host runtime: builds an instrumented variant of
# libpaes_cuda.so (tune/<san>/, host code only -- kernels are unchanged) and
# tests/cpp/stress_threads.cpp against it; `run` executes the stress on the
# GPU and writes gpurun_out/<san>_stress.log.
#   bash scripts/sanitizer_stress.sh build tsan|asan     # here (nvcc, no GPU)
#   bash scripts/sanitizer_stress.sh run tsan|asan       # on the B200 box
set -euo pipefail
cd "$(dirname "$0")/.."
mode="${1:-build}"
san="${2:-tsan}"
case "$san" in
  tsan) flag=thread ;;
  asan) flag=address ;;
  *) echo "sanitizer must be tsan or asan" >&2; exit 2 ;;
esac
dir="tune/$san"
if [ "$mode" = build ]; then
  SAN_FLAG="$flag" SAN_DIR="$dir" python - <<'PY'
import os, sys; sys.path.insert(0, ".")
from paper_1403_7295_b200 import build
build.build(out_lib=os.path.join(os.environ["SAN_DIR"], "libpaes_cuda.so"),
            host_flags=["-fsanitize=" + os.environ["SAN_FLAG"], "-g", "-fno-omit-frame-pointer"])
PY
  /usr/bin/g++ -std=c++17 -O1 -g -fno-omit-frame-pointer -fsanitize="$flag" -Iinclude -I/usr/local/cuda/include \
    tests/cpp/stress_threads.cpp -o "$dir/stress_threads" -L"$dir" -lpaes_cuda -L/usr/local/cuda/lib64 -lcudart \
    -Wl,-rpath,'$ORIGIN' -Wl,-rpath,/usr/local/cuda/lib64
  echo "built $dir/stress_threads"
else
  mkdir -p gpurun_out
  log="gpurun_out/${san}_stress.log"
  # the file jobs' helper threads too: mapped writer + fallocate thread on any
  # file system, detached reclaim of replaced outputs from 4 KiB up
  export PAES_FILE_WRITER="${PAES_FILE_WRITER:-mmap}" PAES_FILE_ASYNC_RECLAIM="${PAES_FILE_ASYNC_RECLAIM:-4096}"
  if [ "$san" = tsan ]; then
    # The CUDA driver's launch path copies kernel parameters into driver-owned
    # buffers under its own synchronisation, which TSAN cannot see; races whose
    # frames are all inside libcuda are suppressed (our frames stay checked).
    printf 'race:libcuda.so\n' > "$dir/suppressions.txt"
    TSAN_OPTIONS="halt_on_error=0 second_deadlock_stack=1 report_signal_unsafe=0 suppressions=$dir/suppressions.txt" \
      "./$dir/stress_threads" 8 40 > "$log" 2>&1 || true
    echo "tsan warnings: $(grep -c 'WARNING: ThreadSanitizer' "$log" || true)"
  else
    # CUDA maps memory inside ASAN's shadow gap; leak checking off (driver-owned
    # allocations live for the process)
    ASAN_OPTIONS="protect_shadow_gap=0 detect_leaks=0 halt_on_error=1" \
      "./$dir/stress_threads" 8 40 > "$log" 2>&1 || true
    echo "asan errors: $(grep -c 'ERROR: AddressSanitizer' "$log" || true)"
  fi
  grep -E "^stress:" "$log" || tail -5 "$log"
fi
