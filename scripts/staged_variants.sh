#!/usr/bin/env bash
# Variant builds of libpaes_cuda.so for the staged-ring A/B (min piece KiB x divisor), into tune/staged_<min>_<div>/.
set -euo pipefail
cd "$(dirname "$0")/.."
for v in "1024 8" "2048 8" "1024 16"; do
  set -- $v
  python - "$1" "$2" <<'PY'
import sys; sys.path.insert(0, ".")
from paper_1403_7295_b200 import build
mn, dv = sys.argv[1], sys.argv[2]
print(build.build(out_lib=f"tune/staged_{mn}_{dv}/libpaes_cuda.so", defines=[f"PAES_STAGED_MIN_KIB={mn}", f"PAES_STAGED_DIV={dv}"]))
PY
done
