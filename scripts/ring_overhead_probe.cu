// Where does a host ring's per-piece cost come from?  1 GiB of pinned host
// data moved host -> device -> host in pieces of p bytes, p = 1 ... 64 MiB:
//   h2d      H2D copies only, one stream
//   copies   H2D then D2H per piece, pieces round-robin over 3 streams (no kernel)
//   copies4  the same over 4 streams
//   nop      + an empty kernel between the copies
//   split_S  one H2D stream, one kernel stream, one D2H stream, S slots, events
//            between them (H2D of piece k+S waits only for D2H of piece k)
//   split_ecb          split_3 with the library's ECB kernel instead of the empty one
//   split_ecb_inplace  ... and the host output written over the host input
//   engine   paes_cuda_chunk (the library's ring, set_pipeline(p, 3)), in place
// GB/s = payload bytes / wall time.  Build: scripts/build_probes.sh
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda_runtime.h>

#include "paes_cuda.h"

#define CK(x)                                                                               \
  do {                                                                                      \
    cudaError_t e_ = (x);                                                                   \
    if (e_ != cudaSuccess) {                                                                \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));            \
      exit(1);                                                                              \
    }                                                                                       \
  } while (0)

__global__ void nop_kernel(unsigned char* p) {
  if (p && threadIdx.x == 1024) p[0] = 0;
}

using clk = std::chrono::steady_clock;

int main() {
  const size_t T = 1ull << 30;
  unsigned char *hin, *hout, *d;
  CK(cudaHostAlloc(reinterpret_cast<void**>(&hin), T + 64, cudaHostAllocDefault));
  CK(cudaHostAlloc(reinterpret_cast<void**>(&hout), T + 64, cudaHostAllocDefault));
  for (size_t i = 0; i < T; i += 4096) hin[i] = static_cast<unsigned char>(i >> 12), hout[i] = 0;
  const int kMaxS = 4;
  const size_t kSlot = 64ull << 20;
  CK(cudaMalloc(&d, kMaxS * kSlot));
  cudaStream_t st[kMaxS];
  for (auto& s : st) CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  unsigned char rk[176];
  unsigned char key[16] = {0};
  if (paes_cuda_expand_key(key, rk) != 0) return 1;

  auto ring = [&](size_t p, int S, bool h2d_only, bool kernel) {
    const size_t n = T / p;
    for (size_t k = 0; k < n; ++k) {
      const int s = static_cast<int>(k % S);
      unsigned char* slot = d + s * kSlot;
      CK(cudaMemcpyAsync(slot, hin + k * p, p, cudaMemcpyHostToDevice, h2d_only ? st[0] : st[s]));
      if (h2d_only) continue;
      if (kernel) nop_kernel<<<148, 512, 0, st[s]>>>(slot);
      CK(cudaMemcpyAsync(hout + k * p, slot, p, cudaMemcpyDeviceToHost, st[s]));
    }
    for (auto& s : st) CK(cudaStreamSynchronize(s));
  };
  cudaStream_t sin, sk, sout;
  CK(cudaStreamCreateWithFlags(&sin, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&sk, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&sout, cudaStreamNonBlocking));
  const int kMaxSplit = 8;
  cudaEvent_t ein[kMaxSplit], ek[kMaxSplit], eout[kMaxSplit];
  for (int i = 0; i < kMaxSplit; ++i) {
    CK(cudaEventCreateWithFlags(&ein[i], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ek[i], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&eout[i], cudaEventDisableTiming));
  }
  unsigned char* dsplit = nullptr;
  // kind 0: empty kernel; 1: the library's ECB encrypt on the slot (in place);
  // 2: ECB with host output == host input (in place on the host too)
  auto split = [&](size_t p, int S, int kind = 0) {
    const size_t n = T / p;
    for (size_t k = 0; k < n; ++k) {
      const int s = static_cast<int>(k % S);
      unsigned char* slot = dsplit + s * p;
      if (k >= static_cast<size_t>(S)) CK(cudaStreamWaitEvent(sin, eout[s], 0));
      CK(cudaMemcpyAsync(slot, hin + k * p, p, cudaMemcpyHostToDevice, sin));
      CK(cudaEventRecord(ein[s], sin));
      CK(cudaStreamWaitEvent(sk, ein[s], 0));
      if (kind == 0) nop_kernel<<<148, 512, 0, sk>>>(slot);
      else if (paes_cuda_ecb_device(PAES_ENCRYPT, slot, slot, p, rk, 0, sk) != 0) exit(1);
      CK(cudaEventRecord(ek[s], sk));
      CK(cudaStreamWaitEvent(sout, ek[s], 0));
      CK(cudaMemcpyAsync((kind == 2 ? hin : hout) + k * p, slot, p, cudaMemcpyDeviceToHost, sout));
      CK(cudaEventRecord(eout[s], sout));
    }
    CK(cudaStreamSynchronize(sout));
    CK(cudaDeviceSynchronize());
  };
  auto time_best = [&](auto&& f) {
    double best = 1e30;
    f();  // warm-up
    for (int r = 0; r < 3; ++r) {
      const auto t0 = clk::now();
      f();
      best = std::min(best, std::chrono::duration<double>(clk::now() - t0).count());
    }
    return T / best / 1e9;
  };
  printf("[\n");
  const size_t ps[] = {1ull << 20, 2ull << 20, 4ull << 20, 8ull << 20, 16ull << 20, 32ull << 20, 64ull << 20};
  for (size_t i = 0; i < sizeof ps / sizeof ps[0]; ++i) {
    const size_t p = ps[i];
    const double h2d = time_best([&] { ring(p, 1, true, false); });
    const double copies = time_best([&] { ring(p, 3, false, false); });
    const double copies4 = time_best([&] { ring(p, 4, false, false); });
    const double nop = time_best([&] { ring(p, 3, false, true); });
    CK(cudaMalloc(&dsplit, kMaxSplit * p));
    const double split3 = time_best([&] { split(p, 3); });
    const double split4 = time_best([&] { split(p, 4); });
    const double split8 = time_best([&] { split(p, 8); });
    const double split_ecb = time_best([&] { split(p, 3, 1); });
    const double split_ecb_inplace = time_best([&] { split(p, 3, 2); });
    CK(cudaFree(dsplit));
    if (paes_cuda_set_pipeline(p, 3) != 0) return 1;
    const double engine = time_best([&] {
      uint64_t olen = 0;
      if (paes_cuda_chunk(PAES_ENCRYPT, hin, T, 0, rk, hin, &olen, 1) != 0) {
        fprintf(stderr, "chunk failed: %s\n", paes_cuda_last_error());
        exit(1);
      }
    });
    printf("  {\"piece_mib\": %zu, \"pieces\": %zu, \"h2d_gbs\": %.2f, \"copies_3s_gbs\": %.2f, \"copies_4s_gbs\": %.2f, "
           "\"copies_nop_kernel_gbs\": %.2f, \"split_3_gbs\": %.2f, \"split_4_gbs\": %.2f, \"split_8_gbs\": %.2f, "
           "\"split_ecb_gbs\": %.2f, \"split_ecb_host_inplace_gbs\": %.2f, \"engine_gbs\": %.2f}%s\n",
           p >> 20, T / p, h2d, copies, copies4, nop, split3, split4, split8, split_ecb, split_ecb_inplace, engine, i + 1 < sizeof ps / sizeof ps[0] ? "," : "");
    fflush(stdout);
  }
  printf("]\n");
  return 0;
}
