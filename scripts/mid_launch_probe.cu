// Fixed cost of one ecb launch at mid sizes (config 1 is 64 MiB): device-side
// time per launch when launches queue back to back, and per call with an
// event pair and a sync around each launch; GB/s and the excess over the
// steady-state rate of the 1 GiB queued case.  Build: scripts/build_probes.sh
#include <cstdio>
#include <cuda_runtime.h>
#include "paes_cuda.h"

int main() {
  unsigned char key[16] = {1}, rk[176];
  paes_cuda_expand_key(key, rk);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  const size_t maxn = 1ull << 30;
  void *din, *dout;
  cudaMalloc(&din, maxn + 64);
  cudaMalloc(&dout, maxn + 64);
  cudaMemset(din, 3, maxn + 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const size_t sizes[] = {16ull << 20, 64ull << 20, 256ull << 20, 1ull << 30};
  printf("[\n");
  for (size_t i = 0; i < 4; ++i) {
    const size_t n = sizes[i];
    const int reps = static_cast<int>(std::max<size_t>(8, (4ull << 30) / n));
    for (int w = 0; w < 3; ++w) paes_cuda_ecb_device(0, din, dout, n, rk, 0, st);
    cudaEventRecord(e0, st);
    for (int r = 0; r < reps; ++r) paes_cuda_ecb_device(0, din, dout, n, rk, 0, st);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double queued_us = 1e3 * ms / reps;
    double best_single = 1e30;
    for (int r = 0; r < 10; ++r) {
      cudaStreamSynchronize(st);
      cudaEventRecord(e0, st);
      paes_cuda_ecb_device(0, din, dout, n, rk, 0, st);
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      best_single = std::min(best_single, 1e3 * ms);
    }
    printf("  {\"bytes\": %zu, \"queued_us\": %.2f, \"queued_gbs\": %.1f, \"single_us\": %.2f, \"single_gbs\": %.1f}%s\n", n,
           queued_us, n / queued_us / 1e3, best_single, n / best_single / 1e3, i < 3 ? "," : "");
  }
  printf("]\n");
  return 0;
}
