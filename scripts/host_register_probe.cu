// Can pageable host buffers be pinned on the fly faster than they can be
// staged?  Times cudaHostRegister / cudaHostUnregister of touched malloc'd
// memory, and the transform of the registered range through paes_cuda_chunk,
// against the staged pageable path.  One JSON line.
// Build: scripts/build_probes.sh
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include <cuda_runtime.h>

#include "paes_cuda.h"

static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

int main() {
  std::uint8_t key[16] = {3}, rk[176];
  paes_cuda_expand_key(key, rk);
  cudaFree(nullptr);
  std::printf("{\"rows\": [");
  bool first = true;
  for (std::size_t n : {16ul << 20, 64ul << 20, 256ul << 20, 1ul << 30}) {
    auto* in = static_cast<std::uint8_t*>(std::malloc(n + 4096));
    auto* out = static_cast<std::uint8_t*>(std::malloc(n + 4096));
    std::memset(in, 7, n + 4096);
    std::memset(out, 0, n + 4096);
    std::uint64_t ol = 0;
    // staged (pageable) path
    paes_cuda_chunk(0, in, n, 0, rk, out, &ol, 1);
    double t = now();
    for (int i = 0; i < 3; ++i) paes_cuda_chunk(0, in, n, 0, rk, out, &ol, 1);
    const double staged = 3.0 * n / (now() - t) / 1e9;
    // register + transform + unregister, per call (unaligned start: +1 page offset +8)
    double reg = 0, unreg = 0, xf = 0;
    int ok = 1;
    for (int i = 0; i < 3; ++i) {
      double a = now();
      ok &= cudaHostRegister(in + 8, n, cudaHostRegisterDefault) == cudaSuccess;
      ok &= cudaHostRegister(out + 8, n, cudaHostRegisterDefault) == cudaSuccess;
      double b = now();
      ok &= paes_cuda_chunk(0, in + 8, n, 0, rk, out + 8, &ol, 1) == PAES_OK;
      double c = now();
      ok &= cudaHostUnregister(in + 8) == cudaSuccess;
      ok &= cudaHostUnregister(out + 8) == cudaSuccess;
      double e = now();
      reg += b - a, xf += c - b, unreg += e - c;
    }
    std::printf("%s{\"bytes\": %zu, \"staged_gbs\": %.2f, \"register_2bufs_gbs\": %.2f, \"transform_registered_gbs\": %.2f, "
                "\"unregister_2bufs_gbs\": %.2f, \"register_transform_unregister_gbs\": %.2f, \"ok\": %d}",
                first ? "" : ", ", n, staged, 3.0 * n / reg / 1e9, 3.0 * n / xf / 1e9, 3.0 * n / unreg / 1e9,
                3.0 * n / (reg + xf + unreg) / 1e9, ok);
    first = false;
    std::free(in);
    std::free(out);
  }
  std::printf("]}\n");
  return 0;
}
