// Concurrent H2D + D2H over pinned memory: does splitting each direction over
// several streams (copy engines) or changing the request granularity lift the
// ~50 GB/s-each-way duplex ceiling the e2e ring runs into?  Copies of 4 GiB
// each way, issued as `pieces` chunks round-robin over `streams` streams per
// direction; best of 3.  Prints one JSON object.  Build: scripts/build_probes.sh
#include <chrono>
#include <cstdio>
#include <vector>

#include <cuda_runtime.h>

int main() {
  const size_t n = 4ull << 30;
  unsigned char *h_in, *h_out, *d_in, *d_out;
  cudaHostAlloc(reinterpret_cast<void**>(&h_in), n, cudaHostAllocDefault);
  cudaHostAlloc(reinterpret_cast<void**>(&h_out), n, cudaHostAllocDefault);
  cudaMalloc(&d_in, n);
  cudaMalloc(&d_out, n);
  for (size_t i = 0; i < n; i += 4096) h_in[i] = 1, h_out[i] = 2;
  std::vector<cudaStream_t> st(16);
  for (auto& s : st) cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  std::printf("{\"rows\": [\n");
  bool first = true;
  const int streams_list[] = {1, 2, 4};
  const size_t piece_list[] = {8ull << 20, 64ull << 20, 256ull << 20};
  for (int mode = 0; mode < 3; ++mode) {  // 0 h2d only, 1 d2h only, 2 both
    for (int ns : streams_list) {
      for (size_t piece : piece_list) {
        double best = 0;
        for (int rep = 0; rep < 3; ++rep) {
          cudaDeviceSynchronize();
          const auto t0 = std::chrono::steady_clock::now();
          size_t k = 0;
          for (size_t off = 0; off < n; off += piece, ++k) {
            const size_t len = std::min(piece, n - off);
            if (mode != 1) cudaMemcpyAsync(d_in + off, h_in + off, len, cudaMemcpyHostToDevice, st[k % ns]);
            if (mode != 0) cudaMemcpyAsync(h_out + off, d_out + off, len, cudaMemcpyDeviceToHost, st[8 + k % ns]);
          }
          cudaDeviceSynchronize();
          const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
          best = std::max(best, n / s / 1e9);
        }
        std::printf("%s  {\"mode\": \"%s\", \"streams_per_dir\": %d, \"piece_mib\": %zu, \"gbs_each_way\": %.2f}",
                    first ? "" : ",\n", mode == 0 ? "h2d" : mode == 1 ? "d2h" : "both", ns, piece >> 20, best);
        first = false;
      }
    }
  }
  std::printf("\n], \"error\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
