// Does a bulk (TMA, cp.async.bulk) copy read pinned HOST memory over PCIe faster than per-thread 128-bit loads?
// The zero-copy route (pinned ranges up to 48 MiB) has the SMs read the caller's buffer with LDG.128 and levels
// off near 40 GB/s with writes in flight; this probe times, on a pinned 256 MiB buffer, 32 and 148 CTAs:
//   ldg_read    host -> device buffer, LDG.128 + STG.128
//   bulk_read   host -> device buffer, cp.async.bulk 16 KiB chunks into shared memory (4 stages), LDS + STG.128
//   ldg_duplex  host -> host (separate pinned buffer), LDG.128 + STG.128
//   bulk_duplex host -> host, bulk loads, STG.128 stores
//   bulk_both   host -> host, bulk loads and bulk stores (cp.async.bulk.global.shared::cta)
// GB/s = bytes read / kernel time (CUDA events), best of 5.  One JSON line.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 scripts/bulk_read_probe.cu -o scripts/bulk_read_probe_bin
#include <cstdint>
#include <cstdio>
#include <cstring>

#include <cuda_runtime.h>

constexpr int kThreads = 512;
constexpr int kChunk = 16 * 1024;  // bytes per bulk copy
constexpr int kStages = 4;

__global__ void __launch_bounds__(kThreads) ldg_copy(const uint4* __restrict__ in, uint4* __restrict__ out, size_t n16) {
  for (size_t i = blockIdx.x * static_cast<size_t>(kThreads) + threadIdx.x; i < n16; i += static_cast<size_t>(gridDim.x) * kThreads) {
    uint4 v = __ldcs(in + i);
    v.x ^= 0x5a5a5a5au;
    __stcs(out + i, v);
  }
}

__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }

template <bool BULK_STORE>
__global__ void __launch_bounds__(kThreads) bulk_copy(const uint8_t* __restrict__ in, uint8_t* __restrict__ out, size_t nchunks) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) unsigned long long bar[kStages];
  uint8_t* stage[kStages];
  for (int s = 0; s < kStages; ++s) stage[s] = sm + s * kChunk;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const size_t first = blockIdx.x, stride = gridDim.x;
  auto issue = [&](size_t c, int s) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(kChunk) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(stage[s])),
                 "l"(in + c * kChunk), "r"(kChunk), "r"(smem_u32(&bar[s]))
                 : "memory");
  };
  // prologue: fill the stages
  if (threadIdx.x == 0) {
    size_t c = first;
    for (int s = 0; s < kStages && c < nchunks; ++s, c += stride) issue(c, s);
  }
  unsigned phase[kStages] = {};
  int s = 0;
  for (size_t c = first; c < nchunks; c += stride, s = (s + 1) % kStages) {
    // wait for the chunk
    unsigned ok = 0;
    while (!ok) {
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(ok)
                   : "r"(smem_u32(&bar[s])), "r"(phase[s])
                   : "memory");
    }
    phase[s] ^= 1;
    uint4* sp = reinterpret_cast<uint4*>(stage[s]);
    if (BULK_STORE) {
      for (int i = threadIdx.x; i < kChunk / 16; i += kThreads) sp[i].x ^= 0x5a5a5a5au;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (threadIdx.x == 0) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + c * kChunk),
                     "r"(smem_u32(stage[s])), "r"(kChunk)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // the stage may be refilled
      }
      __syncthreads();
    } else {
      uint4* op = reinterpret_cast<uint4*>(out + c * kChunk);
      for (int i = threadIdx.x; i < kChunk / 16; i += kThreads) {
        uint4 v = sp[i];
        v.x ^= 0x5a5a5a5au;
        __stcs(op + i, v);
      }
      __syncthreads();  // everyone has read the stage
    }
    const size_t next = c + stride * kStages;
    if (threadIdx.x == 0 && next < nchunks) issue(next, s);
  }
  if (BULK_STORE && threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <class F>
static double best_gbs(F launch, size_t bytes) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  double best = 0;
  for (int rep = 0; rep < 6; ++rep) {
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    if (rep) best = best > bytes / (ms * 1e6) ? best : bytes / (ms * 1e6);
  }
  return best;
}

int main() {
  const size_t n = 256ull << 20;
  uint8_t *hin, *hout, *dbuf;
  cudaHostAlloc(reinterpret_cast<void**>(&hin), n, cudaHostAllocDefault);
  cudaHostAlloc(reinterpret_cast<void**>(&hout), n, cudaHostAllocDefault);
  cudaMalloc(&dbuf, n);
  for (size_t i = 0; i < n; i += 4) {
    const uint32_t v = static_cast<uint32_t>(i * 2654435761u);
    std::memcpy(hin + i, &v, 4);
  }
  cudaFuncSetAttribute(bulk_copy<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kStages * kChunk);
  cudaFuncSetAttribute(bulk_copy<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kStages * kChunk);
  std::printf("{\"bytes\": %zu, \"chunk\": %d, \"stages\": %d", n, kChunk, kStages);
  for (int grid : {32, 148}) {
    const double a = best_gbs([&] { ldg_copy<<<grid, kThreads>>>(reinterpret_cast<const uint4*>(hin), reinterpret_cast<uint4*>(dbuf), n / 16); }, n);
    const double b = best_gbs([&] { bulk_copy<false><<<grid, kThreads, kStages * kChunk>>>(hin, dbuf, n / kChunk); }, n);
    const double c = best_gbs([&] { ldg_copy<<<grid, kThreads>>>(reinterpret_cast<const uint4*>(hin), reinterpret_cast<uint4*>(hout), n / 16); }, n);
    std::memset(hout, 0, n);
    const double d = best_gbs([&] { bulk_copy<false><<<grid, kThreads, kStages * kChunk>>>(hin, hout, n / kChunk); }, n);
    bool ok = true;
    for (size_t i = 0; i < n; i += 4099 * 16) {
      uint32_t x, y;
      std::memcpy(&x, hin + (i & ~size_t(15)), 4);
      std::memcpy(&y, hout + (i & ~size_t(15)), 4);
      ok = ok && (x ^ 0x5a5a5a5au) == y;
    }
    std::memset(hout, 0, n);
    const double e = best_gbs([&] { bulk_copy<true><<<grid, kThreads, kStages * kChunk>>>(hin, hout, n / kChunk); }, n);
    for (size_t i = 0; i < n; i += 4099 * 16) {
      uint32_t x, y;
      std::memcpy(&x, hin + (i & ~size_t(15)), 4);
      std::memcpy(&y, hout + (i & ~size_t(15)), 4);
      ok = ok && (x ^ 0x5a5a5a5au) == y;
    }
    const cudaError_t err = cudaDeviceSynchronize();
    std::printf(", \"grid%d\": {\"ldg_read\": %.2f, \"bulk_read\": %.2f, \"ldg_duplex\": %.2f, \"bulk_duplex\": %.2f, "
                "\"bulk_both\": %.2f, \"check\": \"%s\", \"cuda\": \"%s\"}",
                grid, a, b, c, d, e, ok ? "ok" : "MISMATCH", cudaGetErrorString(err));
  }
  std::printf("}\n");
  return 0;
}
