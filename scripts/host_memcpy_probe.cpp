// Host memory bandwidth on the GPU box: parallel memcpy of 1 GiB (buffers
// pre-faulted) with T threads, alone and as two concurrent teams (the staged
// ring copies pieces in and out at the same time).  GB/s = bytes copied / s
// (each copied byte is one DRAM read + one write).
// Build: g++ -O2 -pthread scripts/host_memcpy_probe.cpp -o scripts/host_memcpy_probe_bin
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

using clk = std::chrono::steady_clock;

static void par_copy(unsigned char* dst, const unsigned char* src, size_t n, unsigned threads) {
  std::vector<std::thread> pool;
  const size_t step = (((n + threads - 1) / threads) + 4095) & ~size_t(4095);
  for (unsigned i = 0; i < threads; ++i) {
    const size_t b = std::min(n, i * step), e = std::min(n, (i + 1) * step);
    if (b < e) pool.emplace_back([=] { std::memcpy(dst + b, src + b, e - b); });
  }
  for (auto& t : pool) t.join();
}

int main() {
  const size_t n = 1ull << 30;
  std::vector<unsigned char*> buf(4);
  for (auto& p : buf) {
    p = static_cast<unsigned char*>(aligned_alloc(4096, n));
    std::memset(p, 1, n);
  }
  const unsigned hw = std::thread::hardware_concurrency();
  printf("{\"hardware_concurrency\": %u, \"rows\": [\n", hw);
  const unsigned ts[] = {1, 2, 4, 8, 12, 16, 24, 32};
  bool first = true;
  for (unsigned t : ts) {
    if (t > 2 * hw) continue;
    double one = 0, two = 0;
    for (int r = 0; r < 3; ++r) {
      auto t0 = clk::now();
      par_copy(buf[1], buf[0], n, t);
      one = std::max(one, n / std::chrono::duration<double>(clk::now() - t0).count() / 1e9);
      t0 = clk::now();
      std::thread a([&] { par_copy(buf[1], buf[0], n, std::max(1u, t / 2)); });
      std::thread b([&] { par_copy(buf[3], buf[2], n, std::max(1u, t / 2)); });
      a.join();
      b.join();
      two = std::max(two, 2.0 * n / std::chrono::duration<double>(clk::now() - t0).count() / 1e9);
    }
    printf("%s  {\"threads\": %u, \"memcpy_gbs\": %.1f, \"two_teams_total_gbs\": %.1f}", first ? "" : ",\n", t, one, two);
    first = false;
  }
  printf("\n]}\n");
  return 0;
}
