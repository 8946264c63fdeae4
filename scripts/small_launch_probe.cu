// Short launches (config 3's small sizes) from a C caller through the C ABI.
// Run it against two library builds (LD_LIBRARY_PATH=<variant dir>) for an
// A/B.  Round 2 tried, and dropped, (a) a compact one-copy table layout for
// short launches (~3.5-way bank conflicts on random data: 1.7-3x slower from
// 1 MiB, within 0.1 us below) and (b) a rolled-loop cipher for the ragged
// tile (less code to fetch cold): neither moves the ~8.2 us single launch
// after an L2 flush nor the ~1.6 us per launch in a graph
// (profiles/r02_small_launch_probe*.json).
//   queued_us : device time per launch, 400 launches queued between one event
//               pair (host-issue bound when the host is slower than the GPU)
//   graph_us  : the same launches captured once in a CUDA graph, replayed
//   flushed_us: one launch after a 256 MiB L2-flushing memset, own events
//   host_us   : host wall time per paes_cuda_ecb_device call
// Prints one JSON object.  Build: scripts/build_probes.sh
#include <chrono>
#include <cstdio>
#include <vector>

#include <cuda_runtime.h>

#include "paes_cuda.h"

static float ev_ms(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main() {
  std::uint8_t key[16] = {9}, rk[176];
  paes_cuda_expand_key(key, rk);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  const size_t maxn = 64ull << 20;
  std::uint8_t *din, *dout, *flush;
  cudaMalloc(&din, maxn + 64);
  cudaMalloc(&dout, maxn + 64);
  cudaMalloc(&flush, 256ull << 20);
  {  // random input: constant bytes would turn every lookup into a broadcast
    std::vector<std::uint8_t> h(maxn + 64);
    std::uint64_t x = 0x9E3779B97F4A7C15ull;
    for (auto& b : h) {
      x ^= x << 13, x ^= x >> 7, x ^= x << 17;
      b = static_cast<std::uint8_t>(x >> 24);
    }
    cudaMemcpy(din, h.data(), h.size(), cudaMemcpyHostToDevice);
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const size_t sizes[] = {16, 1024, 16384, 65536, 262144, 1 << 20, 4 << 20, 16 << 20, 64 << 20};
  const int dirs[] = {0, 1};
  std::printf("{\"rows\": [\n");
  bool first = true;
  // pass 0 warms the host side (CPU clocks, driver caches) and is not printed:
  // the first rows of a cold process read ~1 us slower
  for (int pass = 0; pass < 2; ++pass)
  for (int dir : dirs) {
    for (size_t n : sizes) {
      {
        const int reps = n >= (16u << 20) ? 50 : 400;
        auto call = [&] { return paes_cuda_ecb_device(dir, din, dout, n, rk, 0, st); };
        for (int i = 0; i < 20; ++i) call();
        cudaStreamSynchronize(st);
        // host cost per call (GPU may lag; measured on the issue side)
        auto t0 = std::chrono::steady_clock::now();
        cudaEventRecord(e0, st);
        for (int i = 0; i < reps; ++i) call();
        cudaEventRecord(e1, st);
        auto t1 = std::chrono::steady_clock::now();
        cudaEventSynchronize(e1);
        const double host_us = std::chrono::duration<double, std::micro>(t1 - t0).count() / reps;
        const double queued_us = 1e3 * ev_ms(e0, e1) / reps;
        // graph of `reps` launches
        cudaGraph_t g;
        cudaGraphExec_t ge;
        cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
        for (int i = 0; i < reps; ++i) call();
        cudaStreamEndCapture(st, &g);
        cudaGraphInstantiate(&ge, g, 0);
        cudaGraphLaunch(ge, st);
        cudaStreamSynchronize(st);
        cudaEventRecord(e0, st);
        cudaGraphLaunch(ge, st);
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        const double graph_us = 1e3 * ev_ms(e0, e1) / reps;
        cudaGraphExecDestroy(ge);
        cudaGraphDestroy(g);
        // single launch after an L2 flush
        double fl = 0;
        const int freps = 20;
        for (int i = 0; i < freps; ++i) {
          cudaMemsetAsync(flush, i, 256ull << 20, st);
          cudaEventRecord(e0, st);
          call();
          cudaEventRecord(e1, st);
          cudaEventSynchronize(e1);
          fl += 1e3 * ev_ms(e0, e1);
        }
        const double flushed_us = fl / freps;
        if (pass == 0) continue;
        std::printf("%s  {\"dir\": %d, \"bytes\": %zu, \"host_us\": %.2f, \"queued_us\": %.2f, "
                    "\"graph_us\": %.2f, \"flushed_us\": %.2f, \"flushed_gbs\": %.2f, \"graph_gbs\": %.2f}",
                    first ? "" : ",\n", dir, n, host_us, queued_us, graph_us, flushed_us, n / flushed_us / 1e3,
                    n / graph_us / 1e3);
        first = false;
      }
    }
  }
  std::printf("\n], \"error\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
