// Mid-size pinned e2e (16 MiB .. 1 GiB): would "H2D by the copy engine, then the kernel stores its output
// straight into the pinned host buffer" beat the library's ring (H2D / kernel / D2H on three queues), whose
// last D2H piece runs with nothing to overlap it?  profiles/r01_hybrid_d2h_probe.json measured the idea only
// at 8 GiB with 256 MiB pieces (slower: 44.6 vs 47.2 GB/s).
//   lib     : paes_cuda_chunk on pinned buffers (whatever route the library picks), best of 7
//   hybridP : pieces of P MiB over 3 device buffers; copy stream + kernel stream; best of 7
// GB/s = input bytes / wall time.  One JSON line per size.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I include scripts/hybrid_mid_probe.cu \
//        -L paper_1403_7295_b200/lib -lpaes_cuda -Xlinker -rpath=$PWD/paper_1403_7295_b200/lib -o scripts/hybrid_mid_probe_bin
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <vector>

#include <cuda_runtime.h>

#include "paes_cuda.h"

static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

int main() {
  const std::size_t cap = 1ull << 30;
  std::uint8_t key[16] = {5}, rk[176];
  paes_cuda_expand_key(key, rk);
  std::uint8_t *hin, *hout, *hchk;
  cudaHostAlloc(reinterpret_cast<void**>(&hin), cap + 64, cudaHostAllocDefault);
  cudaHostAlloc(reinterpret_cast<void**>(&hout), cap + 64, cudaHostAllocDefault);
  cudaHostAlloc(reinterpret_cast<void**>(&hchk), cap + 64, cudaHostAllocDefault);
  for (std::size_t i = 0; i < cap; i += 64) hin[i] = static_cast<std::uint8_t>((i >> 6) * 37);
  constexpr int S = 3;
  const std::size_t max_piece = 64ull << 20;
  std::uint8_t* dbuf[S];
  for (auto& p : dbuf) cudaMalloc(&p, max_piece);
  cudaStream_t sc, sk;
  cudaStreamCreateWithFlags(&sc, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&sk, cudaStreamNonBlocking);
  cudaEvent_t copied[S], done[S];
  for (int i = 0; i < S; ++i) {
    cudaEventCreateWithFlags(&copied[i], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming);
    cudaEventRecord(done[i], sk);
  }
  std::uint64_t ol = 0;
  for (std::size_t total : {std::size_t(16) << 20, std::size_t(64) << 20, std::size_t(256) << 20, std::size_t(1) << 30}) {
    double lib = 0;
    for (int rep = 0; rep < 8; ++rep) {
      const double t = now();
      paes_cuda_chunk(0, hin, total, 0, rk, hchk, &ol, 1);
      if (rep) lib = std::max(lib, total / (now() - t) / 1e9);
    }
    std::printf("{\"bytes\": %zu, \"lib_gbs\": %.2f", total, lib);
    for (std::size_t piece : {std::size_t(1) << 20, std::size_t(2) << 20, std::size_t(4) << 20, std::size_t(8) << 20,
                              std::size_t(16) << 20, std::size_t(64) << 20}) {
      if (piece * 2 > total) continue;
      auto hybrid = [&] {
        const std::size_t np = total / piece;
        for (std::size_t k = 0; k < np; ++k) {
          const int b = static_cast<int>(k % S);
          cudaStreamWaitEvent(sc, done[b], 0);  // buffer b free again
          cudaMemcpyAsync(dbuf[b], hin + k * piece, piece, cudaMemcpyHostToDevice, sc);
          cudaEventRecord(copied[b], sc);
          cudaStreamWaitEvent(sk, copied[b], 0);
          paes_cuda_chunk_device(0, dbuf[b], piece, 0, rk, hout + k * piece, &ol, 0, sk);
          cudaEventRecord(done[b], sk);
        }
        cudaStreamSynchronize(sk);
      };
      double best = 0;
      std::memset(hout, 0, total);
      for (int rep = 0; rep < 8; ++rep) {
        const double t = now();
        hybrid();
        if (rep) best = std::max(best, total / (now() - t) / 1e9);
      }
      const bool same = std::memcmp(hout, hchk, total) == 0;
      std::printf(", \"hybrid%zuM_gbs\": %.2f%s", piece >> 20, best, same ? "" : " (MISMATCH)");
    }
    std::printf("}\n");
    std::fflush(stdout);
  }
  return 0;
}
