// Per-call latency of small transforms through the C ABI, against the floor
// of an empty kernel launch + stream sync and a mapped-memory round trip.
// Build: scripts/build_probes.sh
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cuda_runtime.h>

#include "paes_cuda.h"

__global__ void empty_kernel(int* p) {
  if (p && threadIdx.x == 0) *p = 1;
}

__global__ void smem_empty_kernel(int* p) {
  extern __shared__ int sm[];
  if (p && threadIdx.x == 0) sm[0] = *p;
}

// write 128 KiB of smem from a 1 KiB global table, like the T-table staging
__global__ void stage_only_kernel(const unsigned* tab, int* p) {
  extern __shared__ __align__(16) unsigned smu[];
#pragma unroll
  for (int it = 0; it < 16; ++it) {
    const int i = it * 512 + threadIdx.x;
    const unsigned v = tab[(i >> 4) & 255];
    reinterpret_cast<uint4*>(smu)[i] = make_uint4(v, v, v, v);
  }
  __syncthreads();
  if (threadIdx.x == 0 && p) *p = smu[(*p) & 1023];
}

template <class F>
float queued_us(cudaStream_t st, F&& f) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int i = 0; i < 100; ++i) f();
  cudaEventRecord(e0, st);
  for (int i = 0; i < 1000; ++i) f();
  cudaEventRecord(e1, st);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms;  // ms per 1000 launches == us per launch
}

template <class F>
double per_call_us(F&& f, int iters) {
  for (int i = 0; i < 200; ++i) f();
  const auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < iters; ++i) f();
  const auto t1 = std::chrono::steady_clock::now();
  return std::chrono::duration<double, std::micro>(t1 - t0).count() / iters;
}

int main() {
  const int iters = 5000;
  std::uint8_t key[16] = {0}, rk[176];
  paes_cuda_expand_key(key, rk);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  int* dflag;
  cudaMalloc(&dflag, 4);
  std::printf("{\"empty_launch_sync_us\": %.2f", per_call_us([&] {
                empty_kernel<<<1, 32, 0, st>>>(dflag);
                cudaStreamSynchronize(st);
              }, iters));
  std::printf(", \"empty_launch_148x512_sync_us\": %.2f", per_call_us([&] {
                empty_kernel<<<148, 512, 0, st>>>(dflag);
                cudaStreamSynchronize(st);
              }, iters));
  const std::size_t sizes[] = {16, 1031, 4096, 65543, 1048583};
  std::uint8_t *hin, *hout;
  cudaHostAlloc(reinterpret_cast<void**>(&hin), 2 << 20, 0);
  cudaHostAlloc(reinterpret_cast<void**>(&hout), 2 << 20, 0);
  std::vector<std::uint8_t> pin(2 << 20, 7), pout(2 << 20);
  void *din, *dout;
  cudaMalloc(&din, 2 << 20);
  cudaMalloc(&dout, 2 << 20);
  for (std::size_t n : sizes) {
    std::uint64_t ol = 0;
    const double pinned = per_call_us([&] { paes_cuda_chunk(0, hin, n, 1, rk, hout, &ol, 1); }, iters);
    const double pageable = per_call_us([&] { paes_cuda_chunk(0, pin.data(), n, 1, rk, pout.data(), &ol, 1); }, iters);
    const double dev_sync = per_call_us([&] {
      paes_cuda_chunk_device(0, din, n, 1, rk, dout, &ol, 0, st);
      cudaStreamSynchronize(st);
    }, iters);
    // back-to-back async launches: device-side cost per call once host overhead overlaps
    const double dev_async = per_call_us([&] { paes_cuda_chunk_device(0, din, n, 1, rk, dout, &ol, 0, st); }, iters);
    cudaStreamSynchronize(st);
    const double dec_sync = per_call_us([&] {
      std::uint64_t pl = 0;
      paes_cuda_chunk_device(1, dout, ((n / 16) + 1) * 16, 1, rk, din, &pl, 0, st);
    }, iters);
    std::printf(", \"%zu\": {\"host_pinned_us\": %.2f, \"host_pageable_us\": %.2f, \"device_sync_us\": %.2f, "
                "\"device_async_us\": %.2f, \"device_decrypt_final_us\": %.2f}",
                n, pinned, pageable, dev_sync, dev_async, dec_sync);
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  std::uint64_t ol = 0;
  for (int i = 0; i < 100; ++i) paes_cuda_chunk_device(0, din, 1031, 1, rk, dout, &ol, 0, st);
  cudaEventRecord(e0, st);
  for (int i = 0; i < 1000; ++i) paes_cuda_chunk_device(0, din, 1031, 1, rk, dout, &ol, 0, st);
  cudaEventRecord(e1, st);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  std::printf(", \"device_event_1031B_us_per_launch_queued\": %.2f", ms);
  cudaFuncSetAttribute(smem_empty_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  cudaFuncSetAttribute(stage_only_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  unsigned* tab;
  cudaMalloc(&tab, 4096);
  cudaMemset(tab, 1, 4096);
  cudaMemset(dflag, 0, 4);
  std::printf(", \"queued_us\": {\"empty_1x512\": %.2f", queued_us(st, [&] { empty_kernel<<<1, 512, 0, st>>>(dflag); }));
  std::printf(", \"empty_1x512_smem128k\": %.2f",
              queued_us(st, [&] { smem_empty_kernel<<<1, 512, 131072, st>>>(dflag); }));
  std::printf(", \"stage_only_1x512\": %.2f", queued_us(st, [&] { stage_only_kernel<<<1, 512, 131072, st>>>(tab, dflag); }));
  std::printf(", \"stage_only_148x512\": %.2f",
              queued_us(st, [&] { stage_only_kernel<<<148, 512, 131072, st>>>(tab, dflag); }));
  for (std::size_t n : {16ul, 1031ul, 16384ul, 65543ul, 262144ul, 1048583ul})
    std::printf(", \"ecb_%zu\": %.2f", n,
                queued_us(st, [&] { paes_cuda_chunk_device(0, din, n, 1, rk, dout, &ol, 0, st); }));
  std::printf("}}\n");
  return 0;
}
