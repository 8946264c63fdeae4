// Copy-engine throughput vs host/device address alignment: 256 MiB pinned
// H2D and D2H at host offsets {0, 16, 64, 128, 256, 512, 4096+16} with the
// device offset either 0 or equal to the host offset modulo 4096.  Tells the
// ring whether to co-align its device slots with the caller's host pointer.
// One JSON line.  Build: scripts/build_probes.sh
#include <chrono>
#include <cstdio>

#include <cuda_runtime.h>

static double gbs(cudaMemcpyKind kind, void* dst, const void* src, size_t n, cudaStream_t s) {
  cudaMemcpyAsync(dst, src, n, kind, s);
  cudaStreamSynchronize(s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, s);
  for (int i = 0; i < 5; ++i) cudaMemcpyAsync(dst, src, n, kind, s);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return 5.0 * n / (ms / 1e3) / 1e9;
}

int main() {
  const size_t n = 256ull << 20;
  unsigned char *h, *d;
  cudaHostAlloc(reinterpret_cast<void**>(&h), n + 16384, cudaHostAllocDefault);
  cudaMalloc(&d, n + 16384);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  std::printf("{\"bytes\": %zu, \"rows\": [", n);
  bool first = true;
  for (size_t off : {0ul, 16ul, 64ul, 128ul, 256ul, 512ul, 4096ul + 16ul}) {
    const size_t co = off % 4096;
    std::printf("%s{\"host_off\": %zu, \"h2d_dev0\": %.2f, \"h2d_coaligned\": %.2f, \"d2h_dev0\": %.2f, \"d2h_coaligned\": %.2f}",
                first ? "" : ", ", off, gbs(cudaMemcpyHostToDevice, d, h + off, n, s),
                gbs(cudaMemcpyHostToDevice, d + co, h + off, n, s), gbs(cudaMemcpyDeviceToHost, h + off, d, n, s),
                gbs(cudaMemcpyDeviceToHost, h + off, d + co, n, s));
    first = false;
  }
  std::printf("]}\n");
  return 0;
}
