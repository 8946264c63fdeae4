#!/usr/bin/env bash
# Long randomized campaign on the B200: tests/test_gpu_fuzz.py at PAES_FUZZ_SCALE=40 over 8 seeds,
# then tests/cpp/stress_threads.cpp with 16 threads x 400 mixed operations.  Summary: gpurun_out/campaign_summary.txt
set -u
mkdir -p gpurun_out
: > gpurun_out/campaign_summary.txt
for seed in ${FUZZ_SEEDS:-11 12 13 14 15 16 17 18}; do
  PAES_FUZZ_SCALE=40 PAES_FUZZ_SEED=$seed timeout 900 python -m pytest tests/test_gpu_fuzz.py -m gpu -x -q > gpurun_out/campaign_$seed.log 2>&1
  echo "fuzz seed=$seed scale=40 rc=$? $(tail -1 gpurun_out/campaign_$seed.log)" >> gpurun_out/campaign_summary.txt
done
g++ -std=c++17 -O2 -Iinclude -I/usr/local/cuda/include tests/cpp/stress_threads.cpp -o /tmp/stress_threads \
  -Lpaper_1403_7295_b200/lib -lpaes_cuda -L/usr/local/cuda/lib64 -lcudart \
  -Wl,-rpath,$PWD/paper_1403_7295_b200/lib -Wl,-rpath,/usr/local/cuda/lib64
timeout 1200 /tmp/stress_threads 16 400 > gpurun_out/campaign_stress.log 2>&1
echo "stress 16x400 rc=$? $(tail -1 gpurun_out/campaign_stress.log)" >> gpurun_out/campaign_summary.txt
