// Many host threads issuing short host-pointer calls at once (a server
// encrypting small messages on every worker thread, or the reference's
// threaded strategy over small chunks): aggregate calls/s and GB/s of
// paes_cuda_chunk (encrypt, always-pad, final) from T threads, each on its own
// buffers, for pinned (zero-copy kernel path) and pageable (mapped bounce
// buffer) memory.  Every output is checked against a single-threaded call.
// Run it against two library builds (LD_LIBRARY_PATH=<variant dir>) for an A/B.
// One JSON line.  Build: scripts/build_probes.sh
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include "paes_cuda.h"

static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

int main(int argc, char** argv) {
  const double secs = argc > 1 ? std::atof(argv[1]) : 1.0;
  std::uint8_t key[16] = {7}, rk[176];
  paes_cuda_expand_key(key, rk);
  cudaFree(nullptr);
  std::printf("{\"rows\": [");
  bool first = true;
  for (int pinned : {1, 0}) {
    for (std::size_t n : {4096ul, 65536ul}) {
      const std::size_t out_n = (n / 16 + 1) * 16;
      // reference output from one call
      std::vector<std::uint8_t> src(n), want(out_n);
      for (std::size_t i = 0; i < n; ++i) src[i] = static_cast<std::uint8_t>(i * 131 + 7);
      std::uint64_t ol = 0;
      paes_cuda_chunk(PAES_ENCRYPT, src.data(), n, 1, rk, want.data(), &ol, 1);
      for (int T : {1, 2, 4, 8, 16}) {
        std::atomic<long> calls{0}, bad{0};
        std::atomic<bool> go{false}, stop{false};
        std::vector<std::thread> th;
        for (int t = 0; t < T; ++t) {
          th.emplace_back([&, t] {
            std::uint8_t *in, *out;
            if (pinned) {
              cudaHostAlloc(reinterpret_cast<void**>(&in), n, 0);
              cudaHostAlloc(reinterpret_cast<void**>(&out), out_n, 0);
            } else {
              in = static_cast<std::uint8_t*>(std::malloc(n));
              out = static_cast<std::uint8_t*>(std::malloc(out_n));
            }
            std::memcpy(in, src.data(), n);
            std::uint64_t len = 0;
            for (int w = 0; w < 20; ++w) paes_cuda_chunk(PAES_ENCRYPT, in, n, 1, rk, out, &len, 1);
            while (!go.load()) std::this_thread::yield();
            long c = 0;
            while (!stop.load(std::memory_order_relaxed)) {
              std::memset(out, 0, 16);
              if (paes_cuda_chunk(PAES_ENCRYPT, in, n, 1, rk, out, &len, 1) != PAES_OK || len != out_n ||
                  std::memcmp(out, want.data(), out_n) != 0)
                bad.fetch_add(1);
              ++c;
            }
            calls.fetch_add(c);
            if (pinned) {
              cudaFreeHost(in);
              cudaFreeHost(out);
            } else {
              std::free(in);
              std::free(out);
            }
            (void)t;
          });
        }
        std::this_thread::sleep_for(std::chrono::milliseconds(200));
        const double t0 = now();
        go.store(true);
        std::this_thread::sleep_for(std::chrono::duration<double>(secs));
        stop.store(true);
        for (auto& x : th) x.join();
        const double el = now() - t0;
        const double cps = calls.load() / el;
        std::printf("%s{\"pinned\": %d, \"bytes\": %zu, \"threads\": %d, \"calls_per_s\": %.0f, \"us_per_call\": %.2f, "
                    "\"gbs\": %.3f, \"bad\": %ld}",
                    first ? "" : ", ", pinned, n, T, cps, 1e6 / cps * T, cps * n / 1e9, bad.load());
        first = false;
        std::fflush(stdout);
      }
    }
  }
  std::printf("], \"error\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
