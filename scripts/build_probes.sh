#!/usr/bin/env bash
# Build the C/CUDA probes in scripts/ against the in-tree libpaes_cuda.so
# (run __graft_entry__.build() first).  Binaries land next to their sources
# as scripts/<name>_bin (git-ignored; they travel to the GPU box with gpurun).
set -euo pipefail
cd "$(dirname "$0")/.."
for src in scripts/small_latency.cu scripts/zero_copy_probe.cu scripts/host_register_probe.cu \
           scripts/registered_zero_copy_probe.cu scripts/hybrid_d2h_probe.cu scripts/copy_align_probe.cu scripts/lookup_path_probe.cu \
           scripts/ring_overhead_probe.cu scripts/mid_launch_probe.cu scripts/small_launch_probe.cu scripts/pcie_streams_probe.cu \
           scripts/thp_register_probe.cu scripts/flush_floor_probe.cu scripts/concurrent_small_probe.cu scripts/sync_latency_probe.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O2 -ccbin /usr/bin/g++ -I include "$src" \
       -L paper_1403_7295_b200/lib -lpaes_cuda -Xlinker -rpath='$ORIGIN/../paper_1403_7295_b200/lib' \
       -o "${src%.cu}_bin"
done
echo "built: $(ls scripts/*_bin | tr '\n' ' ')"
