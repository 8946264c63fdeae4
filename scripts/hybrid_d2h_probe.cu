// Can the kernel's own stores replace the D2H copy engine on the e2e path?
//   ce_d2h   : cudaMemcpyAsync device -> pinned host
//   sm_d2h   : ecb kernel reading device memory, writing pinned host (UVA)
//   ring     : paes_cuda_chunk on pinned buffers, copy-engine ring (zero-copy off)
//   hybrid   : per piece, H2D by copy engine, then the kernel writes its output
//              straight into the pinned host buffer; pieces double-buffered
// GB/s = input bytes / wall time.  One JSON line.
// Build: scripts/build_probes.sh
#include <chrono>
#include <cstdio>
#include <cstring>
#include <vector>

#include <cuda_runtime.h>

#include "paes_cuda.h"

static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

int main() {
  const std::size_t total = 8ull << 30, piece = 256ull << 20;
  std::uint8_t key[16] = {5}, rk[176];
  paes_cuda_expand_key(key, rk);
  std::uint8_t *hin, *hout, *hchk;
  cudaHostAlloc(reinterpret_cast<void**>(&hin), total, cudaHostAllocDefault);
  cudaHostAlloc(reinterpret_cast<void**>(&hout), total, cudaHostAllocDefault);
  cudaHostAlloc(reinterpret_cast<void**>(&hchk), total, cudaHostAllocDefault);
  for (std::size_t i = 0; i < total; i += 4096) hin[i] = static_cast<std::uint8_t>(i >> 12);
  std::uint8_t* dbuf[2];
  cudaMalloc(&dbuf[0], piece);
  cudaMalloc(&dbuf[1], piece);
  cudaStream_t sc, sk;
  cudaStreamCreateWithFlags(&sc, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&sk, cudaStreamNonBlocking);
  std::uint64_t ol = 0;

  // ce_d2h / sm_d2h on 1 GiB
  const std::size_t one = 1ull << 30;
  std::uint8_t* dbig;
  cudaMalloc(&dbig, one);
  cudaMemcpy(dbig, hin, one, cudaMemcpyHostToDevice);
  double t = now();
  for (int i = 0; i < 3; ++i) cudaMemcpyAsync(hout, dbig, one, cudaMemcpyDeviceToHost, sc);
  cudaStreamSynchronize(sc);
  const double ce_d2h = 3.0 * one / (now() - t) / 1e9;
  paes_cuda_chunk_device(0, dbig, one, 0, rk, hout, &ol, 0, sk);
  cudaStreamSynchronize(sk);
  t = now();
  for (int i = 0; i < 3; ++i) paes_cuda_chunk_device(0, dbig, one, 0, rk, hout, &ol, 0, sk);
  cudaStreamSynchronize(sk);
  const double sm_d2h = 3.0 * one / (now() - t) / 1e9;
  cudaFree(dbig);

  // ring
  paes_cuda_set_zero_copy_max(0);
  paes_cuda_chunk(0, hin, total, 0, rk, hchk, &ol, 1);
  t = now();
  paes_cuda_chunk(0, hin, total, 0, rk, hchk, &ol, 1);
  const double ring = total / (now() - t) / 1e9;

  // hybrid
  cudaEvent_t copied[2], done[2];
  for (int i = 0; i < 2; ++i) {
    cudaEventCreateWithFlags(&copied[i], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming);
    cudaEventRecord(done[i], sk);
  }
  auto hybrid = [&] {
    const std::size_t np = total / piece;
    for (std::size_t k = 0; k < np; ++k) {
      const int b = static_cast<int>(k & 1);
      cudaStreamWaitEvent(sc, done[b], 0);  // buffer b free again
      cudaMemcpyAsync(dbuf[b], hin + k * piece, piece, cudaMemcpyHostToDevice, sc);
      cudaEventRecord(copied[b], sc);
      cudaStreamWaitEvent(sk, copied[b], 0);
      paes_cuda_chunk_device(0, dbuf[b], piece, 0, rk, hout + k * piece, &ol, 0, sk);
      cudaEventRecord(done[b], sk);
    }
    cudaStreamSynchronize(sk);
  };
  hybrid();
  t = now();
  hybrid();
  const double hyb = total / (now() - t) / 1e9;
  const bool same = std::memcmp(hout, hchk, total) == 0;
  std::printf("{\"ce_d2h_gbs\": %.2f, \"sm_d2h_gbs\": %.2f, \"ring_8GiB_gbs\": %.2f, \"hybrid_8GiB_gbs\": %.2f, "
              "\"identical\": %s}\n",
              ce_d2h, sm_d2h, ring, hyb, same ? "true" : "false");
  return 0;
}
