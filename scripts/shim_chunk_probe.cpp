// The C++ drop-in (include/paes_gpu.hpp: paes::gpu::encrypt_chunk / decrypt_chunk, the reference's
// exec.hpp:61-65 signatures) on large std::vector inputs: seconds and GB/s per call, result checked by
// round trip.  Build twice to A/B the untouched result vector (paes_gpu.hpp detail::result_bytes):
//   g++ -std=c++20 -O2 -Iinclude scripts/shim_chunk_probe.cpp -o /tmp/shim_probe -Lpaper_1403_7295_b200/lib -lpaes_cuda
//       -Wl,-rpath,$PWD/paper_1403_7295_b200/lib                       (result pages first touched by the engine)
//   g++ ... -DPAES_GPU_NO_UNINIT -o /tmp/shim_probe_zero                (std::vector<uint8_t>(n): zero-filled first)
//   /tmp/shim_probe [bytes ...]
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

#include "paes_gpu.hpp"

static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

int main(int argc, char** argv) {
  std::vector<std::size_t> sizes;
  for (int i = 1; i < argc; ++i) sizes.push_back(std::strtoull(argv[i], nullptr, 10));
  if (sizes.empty()) sizes = {std::size_t(64) << 20, std::size_t(1) << 30, std::size_t(4) << 30};
  paes::gpu::Key128 key{};
  for (int i = 0; i < 16; ++i) key.bytes[i] = static_cast<std::uint8_t>(i * 7 + 1);
  const paes::gpu::RoundKeySchedule ks(key);
#ifdef PAES_GPU_NO_UNINIT
  const char* mode = "zero_filled_vector";
#else
  const char* mode = "untouched_vector";
#endif
  std::printf("{\"mode\": \"%s\"", mode);
  for (std::size_t n : sizes) {
    std::vector<std::uint8_t> pt(n + 7);
    std::mt19937_64 rng(n);
    for (std::size_t i = 0; i + 8 <= pt.size(); i += 8) {
      const std::uint64_t v = rng();
      std::memcpy(pt.data() + i, &v, 8);
    }
    double enc = 1e9, dec = 1e9;
    bool ok = true;
    for (int rep = 0; rep < 4; ++rep) {  // rep 0 warms the context and the rings
      double t = now();
      std::vector<std::uint8_t> ct = paes::gpu::encrypt_chunk(pt, true, ks);
      const double e = now() - t;
      t = now();
      std::vector<std::uint8_t> back = paes::gpu::decrypt_chunk(ct, true, ks);
      const double d = now() - t;
      ok = ok && ct.size() == (pt.size() / 16 + 1) * 16 && back == pt;
      if (rep) enc = std::min(enc, e), dec = std::min(dec, d);
    }
    std::printf(", \"%zu\": {\"encrypt_s\": %.4f, \"encrypt_gbs\": %.2f, \"decrypt_s\": %.4f, \"decrypt_gbs\": %.2f, \"round_trip\": \"%s\"}",
                pt.size(), enc, pt.size() / enc / 1e9, dec, pt.size() / dec / 1e9, ok ? "ok" : "MISMATCH");
    std::fflush(stdout);
  }
  std::printf("}\n");
  return 0;
}
