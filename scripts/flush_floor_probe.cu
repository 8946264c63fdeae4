// The floor under config 3's "flushed" rows: one launch timed by its own
// event pair right after a 256 MiB L2-flushing memset (the bench rule for
// inputs smaller than L2).  Compares an empty kernel (1 CTA and 148 CTAs of
// 512 threads, no PDL) with paes_cuda_ecb_device at 16 B / 1 KiB / 64 KiB,
// and the same calls without the flush (back-to-back event pairs, L2 warm).
// If the empty kernel already costs most of the ~8 us, the rows measure the
// launch after a flush, not the cipher.  One JSON line.
// Build: scripts/build_probes.sh
#include <cstdint>
#include <cstdio>

#include <cuda_runtime.h>

#include "paes_cuda.h"

__global__ void empty_kernel() {}

int main() {
  std::uint8_t key[16] = {9}, rk[176];
  paes_cuda_expand_key(key, rk);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  std::uint8_t *din, *dout, *flush;
  cudaMalloc(&din, 1 << 20);
  cudaMalloc(&dout, 1 << 20);
  cudaMemset(din, 0x5a, 1 << 20);
  cudaMalloc(&flush, 256ull << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timed = [&](auto call, bool do_flush) {
    const int reps = 30;
    double total = 0;
    for (int i = 0; i < reps + 3; ++i) {
      if (do_flush) cudaMemsetAsync(flush, i, 256ull << 20, st);
      cudaEventRecord(e0, st);
      call();
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      if (i >= 3) total += ms;
    }
    return 1e3 * total / reps;
  };
  std::printf("{\"rows\": [");
  bool first = true;
  auto row = [&](const char* name, auto call) {
    const double fl = timed(call, true), warm = timed(call, false);
    std::printf("%s{\"case\": \"%s\", \"flushed_us\": %.2f, \"warm_us\": %.2f}", first ? "" : ", ", name, fl, warm);
    first = false;
  };
  row("empty 1x512", [&] { empty_kernel<<<1, 512, 0, st>>>(); });
  row("empty 148x512", [&] { empty_kernel<<<148, 512, 0, st>>>(); });
  for (size_t n : {16ul, 1024ul, 65536ul}) {
    char name[64];
    std::snprintf(name, sizeof name, "ecb_device encrypt %zu B", n);
    row(name, [&] { paes_cuda_ecb_device(0, din, dout, n, rk, 0, st); });
  }
  std::printf("], \"error\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
