// Pinned host -> pinned host transform: copy-engine pipeline (paes_cuda_chunk
// with zero-copy disabled) against one zero-copy kernel that reads and writes the host buffers over
// PCIe through their UVA device pointers (paes_cuda_chunk_device on host
// pointers).  Prints one JSON line; GB/s = input bytes / wall time per call.
// Build: scripts/build_probes.sh
#include <chrono>
#include <cstdio>
#include <cstring>

#include <cuda_runtime.h>

#include "paes_cuda.h"

template <class F>
double gbs(std::size_t n, F&& f) {
  f();
  f();
  int iters = static_cast<int>(std::max<std::size_t>(3, std::min<std::size_t>(2000, (2ull << 30) / std::max<std::size_t>(n, 1))));
  const auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < iters; ++i) f();
  const auto t1 = std::chrono::steady_clock::now();
  const double s = std::chrono::duration<double>(t1 - t0).count() / iters;
  return n / s / 1e9;
}

int main() {
  const std::size_t maxn = 1ull << 30;
  std::uint8_t key[16] = {1}, rk[176];
  paes_cuda_expand_key(key, rk);
  std::uint8_t *hin, *hout, *hchk;
  cudaHostAlloc(reinterpret_cast<void**>(&hin), maxn + 64, cudaHostAllocPortable | cudaHostAllocMapped);
  cudaHostAlloc(reinterpret_cast<void**>(&hout), maxn + 64, cudaHostAllocPortable | cudaHostAllocMapped);
  cudaHostAlloc(reinterpret_cast<void**>(&hchk), maxn + 64, cudaHostAllocPortable | cudaHostAllocMapped);
  for (std::size_t i = 0; i < maxn; i += 4096) hin[i] = static_cast<std::uint8_t>(i >> 12);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  std::printf("{\"rows\": [");
  bool first = true;
  for (std::size_t n : {65536ul, 262144ul, 1ul << 20, 4ul << 20, 16ul << 20, 64ul << 20, 256ul << 20, 1ul << 30}) {
    std::uint64_t ol = 0;
    paes_cuda_set_zero_copy_max(0);  // force the copy-engine ring
    const double ce = gbs(n, [&] { paes_cuda_chunk(0, hin, n, 0, rk, hout, &ol, 1); });
    paes_cuda_set_zero_copy_max(128ull << 20);
    const double zc = gbs(n, [&] {
      paes_cuda_chunk_device(0, hin, n, 0, rk, hchk, &ol, 0, st);
      cudaStreamSynchronize(st);
    });
    const bool same = std::memcmp(hout, hchk, n) == 0;
    std::printf("%s{\"bytes\": %zu, \"copy_engine_gbs\": %.2f, \"zero_copy_gbs\": %.2f, \"identical\": %s}",
                first ? "" : ", ", n, ce, zc, same ? "true" : "false");
    first = false;
  }
  std::printf("]}\n");
  return 0;
}
