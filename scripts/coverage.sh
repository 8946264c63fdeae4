#!/usr/bin/env bash
# Host-side line coverage of the runtime under the whole test suite.
#   bash scripts/coverage.sh build     # here: gcov-instrumented variant in tune/cov (kernels unchanged)
#   bash scripts/coverage.sh run       # on the B200: both suites against it, .gcda under gpurun_out/gcov
#   bash scripts/coverage.sh report    # here: per-file line coverage (gpurun_out/coverage.txt)
set -euo pipefail
cd "$(dirname "$0")/.."
case "${1:-build}" in
  build)
    python - <<'PY'
import os, subprocess, sys
sys.path.insert(0, ".")
from paper_1403_7295_b200 import build as b
out = os.path.abspath("tune/cov")
os.makedirs(out, exist_ok=True)
objs = []
for src in b.SOURCES:
    obj = os.path.join(out, src + ".o")
    cmd = [b.NVCC] + b.CCBIN + b.ARCH + b.FLAGS + ["-Xcompiler", "--coverage,-O0", "-c", os.path.join(b.CSRC, src), "-o", obj]
    subprocess.run(cmd, check=True, capture_output=True)
    objs.append(obj)
subprocess.run([b.NVCC] + b.CCBIN + b.ARCH + ["-Xcompiler", "--coverage", "-shared", "-o", os.path.join(out, "libpaes_cuda.so")]
               + objs + ["-lpthread", "-lgcov"], check=True, capture_output=True)
print("built", out)
PY
    ;;
  run)
    export PAES_CUDA_LIB="$PWD/tune/cov/libpaes_cuda.so" GCOV_PREFIX="$PWD/gpurun_out/gcov" GCOV_PREFIX_STRIP=0
    python -m pytest tests -m gpu -q > gpurun_out/cov_gpu.log 2>&1; echo "gpu rc=$?"
    python -m pytest tests -m "not gpu" -q > gpurun_out/cov_cpu.log 2>&1; echo "cpu rc=$?"
    ;;
  report)
    cp gpurun_out/gcov"$PWD"/tune/cov/*.gcda tune/cov/
    (cd tune/cov && for f in runtime.cu abi_core.cu abi_batch.cu abi_file.cu host_rules.cpp; do
       gcov -o . -n "$f.o" 2>/dev/null | grep -A1 "File '.*csrc/$f'"; done) | tee gpurun_out/coverage.txt
    ;;
esac
