// A/B of the library's hybrid route (runtime.cu run_host_range_hybrid: copy-engine H2D + kernel stores into the
// pinned output) against the copy-engine ring, through the public call: paes_cuda_chunk on pinned buffers with
// PAES_HYBRID=0 / 1 (read per call), separate in/out buffers and in place, encrypt (always-pad) and final decrypt.
// GB/s = input bytes / wall time, best of 9 after a warm call; outputs of both routes compared byte for byte.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I include scripts/hybrid_route_ab.cu \
//        -L paper_1403_7295_b200/lib -lpaes_cuda -Xlinker -rpath=$PWD/paper_1403_7295_b200/lib -o scripts/hybrid_route_ab_bin
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include <cuda_runtime.h>

#include "paes_cuda.h"

static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

int main() {
  const std::size_t cap = (1ull << 30) + 64;
  std::uint8_t key[16] = {9, 1, 7}, rk[176];
  paes_cuda_expand_key(key, rk);
  std::uint8_t *hin, *ha, *hb;
  cudaHostAlloc(reinterpret_cast<void**>(&hin), cap, cudaHostAllocDefault);
  cudaHostAlloc(reinterpret_cast<void**>(&ha), cap, cudaHostAllocDefault);
  cudaHostAlloc(reinterpret_cast<void**>(&hb), cap, cudaHostAllocDefault);
  for (std::size_t i = 0; i < cap; i += 8) {
    const std::uint64_t v = i * 0x9e3779b97f4a7c15ull;
    std::memcpy(hin + i, &v, 8);
  }
  std::uint64_t ol = 0;
  for (std::size_t mib : {40, 49, 64, 96, 128, 256, 512, 768}) {
    const std::size_t n = (mib << 20) + 7;
    double gbs[2][3] = {};
    std::uint64_t olen[2] = {};
    bool ok = true;
    for (int hyb = 0; hyb < 2; ++hyb) {
      ::setenv("PAES_HYBRID", hyb ? "1" : "0", 1);
      std::uint8_t* out = hyb ? hb : ha;
      for (int rep = 0; rep < 10; ++rep) {  // encrypt, separate buffers
        const double t = now();
        if (paes_cuda_chunk(0, hin, n, 1, rk, out, &ol, 1) != 0) ok = false;
        if (rep) gbs[hyb][0] = std::max(gbs[hyb][0], n / (now() - t) / 1e9);
      }
      olen[hyb] = ol;
    }
    ok = ok && olen[0] == olen[1] && std::memcmp(ha, hb, olen[0]) == 0;
    for (int hyb = 0; hyb < 2; ++hyb) {
      ::setenv("PAES_HYBRID", hyb ? "1" : "0", 1);
      std::uint8_t* buf = hyb ? hb : ha;  // holds the ciphertext
      for (int rep = 0; rep < 10; ++rep) {  // final decrypt in place, then encrypt in place again
        double t = now();
        if (paes_cuda_chunk(1, buf, olen[0], 1, rk, buf, &ol, 1) != 0 || ol != n) ok = false;
        if (rep) gbs[hyb][1] = std::max(gbs[hyb][1], olen[0] / (now() - t) / 1e9);
        if (std::memcmp(buf, hin, 4096) != 0 || std::memcmp(buf + n - 4096, hin + n - 4096, 4096) != 0) ok = false;
        t = now();
        if (paes_cuda_chunk(0, buf, n, 1, rk, buf, &ol, 1) != 0 || ol != olen[0]) ok = false;
        if (rep) gbs[hyb][2] = std::max(gbs[hyb][2], n / (now() - t) / 1e9);
      }
    }
    ok = ok && std::memcmp(ha, hb, olen[0]) == 0;
    std::printf("{\"MiB\": %zu, \"ring\": {\"enc\": %.2f, \"dec_inplace\": %.2f, \"enc_inplace\": %.2f}, "
                "\"hybrid\": {\"enc\": %.2f, \"dec_inplace\": %.2f, \"enc_inplace\": %.2f}, \"identical\": %s}\n",
                mib, gbs[0][0], gbs[0][1], gbs[0][2], gbs[1][0], gbs[1][1], gbs[1][2], ok ? "true" : "false");
    std::fflush(stdout);
  }
  return 0;
}
