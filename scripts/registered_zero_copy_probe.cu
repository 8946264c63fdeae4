// Zero-copy on cudaHostRegister'ed malloc memory vs cudaHostAlloc memory:
// flags reported by cudaHostGetFlags, and per-call throughput of repeated
// transforms (zero-copy route vs copy ring) on the same registered buffer.
// Build: scripts/build_probes.sh
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include <cuda_runtime.h>

#include "paes_cuda.h"

static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

int main() {
  std::uint8_t key[16] = {3}, rk[176];
  paes_cuda_expand_key(key, rk);
  const std::size_t n = 64ul << 20;
  std::printf("{");
  for (unsigned rflags : {0u, 2u}) {  // cudaHostRegisterDefault, cudaHostRegisterMapped
    auto* in = static_cast<std::uint8_t*>(std::malloc(n + 4096));
    auto* out = static_cast<std::uint8_t*>(std::malloc(n + 4096));
    std::memset(in, 1, n + 4096);
    std::memset(out, 0, n + 4096);
    cudaHostRegister(in, n + 4096, rflags);
    cudaHostRegister(out, n + 4096, rflags);
    unsigned fl = 99;
    const int rc = static_cast<int>(cudaHostGetFlags(&fl, in + 100));
    cudaGetLastError();
    std::printf("%s\"register_flags_%u\": {\"getflags_rc\": %d, \"flags\": %u, \"zero_copy_gbs\": [", rflags ? ", " : "",
                rflags, rc, fl);
    std::uint64_t ol;
    for (int i = 0; i < 5; ++i) {
      const double t = now();
      paes_cuda_chunk(0, in, n, 0, rk, out, &ol, 1);
      std::printf("%s%.2f", i ? ", " : "", n / (now() - t) / 1e9);
    }
    std::printf("], \"ring_gbs\": [");
    paes_cuda_set_zero_copy_max(0);
    for (int i = 0; i < 3; ++i) {
      const double t = now();
      paes_cuda_chunk(0, in, n, 0, rk, out, &ol, 1);
      std::printf("%s%.2f", i ? ", " : "", n / (now() - t) / 1e9);
    }
    paes_cuda_set_zero_copy_max(128ull << 20);
    std::printf("]}");
    cudaHostUnregister(in);
    cudaHostUnregister(out);
    std::free(in);
    std::free(out);
  }
  std::uint8_t *a0, *a1;
  cudaHostAlloc(reinterpret_cast<void**>(&a0), n + 4096, cudaHostAllocDefault);
  cudaHostAlloc(reinterpret_cast<void**>(&a1), n + 4096, cudaHostAllocDefault);
  unsigned fl = 99;
  cudaHostGetFlags(&fl, a0 + 100);
  std::printf(", \"hostalloc_default\": {\"flags\": %u, \"zero_copy_gbs\": [", fl);
  std::uint64_t ol;
  for (int i = 0; i < 3; ++i) {
    const double t = now();
    paes_cuda_chunk(0, a0, n, 0, rk, a1, &ol, 1);
    std::printf("%s%.2f", i ? ", " : "", n / (now() - t) / 1e9);
  }
  std::printf("]}}\n");
  return 0;
}
