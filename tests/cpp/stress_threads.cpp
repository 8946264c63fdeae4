// Multi-threaded stress of every host-side entry point of libpaes_cuda.so,
// for ThreadSanitizer runs (scripts/tsan_stress.sh) and as a plain stress
// test.  Threads mix: pageable and pinned chunk transforms, the zero-copy
// route, device-pointer transforms on private streams, host batches, file
// jobs, state transforms and runtime reconfiguration.  Every result is
// checked by round trip; exit code = number of failures.
#include <unistd.h>

#include <atomic>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include "paes_cuda.h"

static std::atomic<int> g_fail{0};

#define EXPECT(c, what)                                                                   \
  do {                                                                                    \
    if (!(c)) {                                                                           \
      std::fprintf(stderr, "FAIL %s (%s:%d): %s\n", what, __FILE__, __LINE__, paes_cuda_last_error()); \
      g_fail.fetch_add(1);                                                                \
    }                                                                                     \
  } while (0)

static void fill(std::vector<std::uint8_t>& v, std::mt19937_64& rng) {
  for (auto& x : v) x = static_cast<std::uint8_t>(rng());
}

static void worker(int id, int iters) {
  std::mt19937_64 rng(1000 + id);
  std::uint8_t key[16], rk[176];
  for (auto& k : key) k = static_cast<std::uint8_t>(rng());
  paes_cuda_expand_key(key, rk);
  cudaSetDevice(0);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  for (int it = 0; it < iters; ++it) {
    const int op = static_cast<int>(rng() % 7);
    const std::uint64_t n = (rng() % 4 == 0) ? (rng() % (6u << 20)) : (rng() % 70000);
    std::vector<std::uint8_t> data(n), ct(n + 16), back(n + 16);
    fill(data, rng);
    std::uint64_t m = 0, k = 0;
    switch (op) {
      case 0: {  // pageable host chunk round trip; 3 explicit shards (the shard pool) or the auto rule
        const int ng = (rng() % 2) ? 3 : 0;
        EXPECT(paes_cuda_chunk(0, data.data(), n, 1, rk, ct.data(), &m, ng) == 0, "pageable encrypt");
        EXPECT(paes_cuda_chunk(1, ct.data(), m, 1, rk, back.data(), &k, ng) == 0, "pageable decrypt");
        EXPECT(k == n && std::memcmp(back.data(), data.data(), n) == 0, "pageable round trip");
        break;
      }
      case 1: {  // pinned host chunk (zero-copy route or ring, whichever applies)
        std::uint8_t *a = nullptr, *b = nullptr;
        cudaHostAlloc(reinterpret_cast<void**>(&a), n + 64, cudaHostAllocDefault);
        cudaHostAlloc(reinterpret_cast<void**>(&b), n + 64, cudaHostAllocDefault);
        std::memcpy(a + 16, data.data(), n);
        EXPECT(paes_cuda_chunk(0, a + 16, n, 1, rk, b, &m, 1) == 0, "pinned encrypt");
        EXPECT(paes_cuda_chunk(1, b, m, 1, rk, a, &k, 1) == 0, "pinned decrypt");
        EXPECT(k == n && std::memcmp(a, data.data(), n) == 0, "pinned round trip");
        cudaFreeHost(a);
        cudaFreeHost(b);
        break;
      }
      case 2: {  // device pointers on a private stream
        std::uint8_t *d = nullptr, *e = nullptr;
        cudaMalloc(&d, n + 32);
        cudaMalloc(&e, n + 32);
        cudaMemcpyAsync(d, data.data(), n, cudaMemcpyHostToDevice, st);
        EXPECT(paes_cuda_chunk_device(0, d, n, 1, rk, e, &m, 0, st) == 0, "device encrypt");
        EXPECT(paes_cuda_chunk_device(1, e, m, 1, rk, d, &k, 0, st) == 0, "device decrypt");
        cudaMemcpyAsync(back.data(), d, n, cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        EXPECT(k == n && std::memcmp(back.data(), data.data(), n) == 0, "device round trip");
        cudaFree(d);
        cudaFree(e);
        break;
      }
      case 3: {  // host batch of small messages, per-message keys
        const std::uint32_t nm = 1 + static_cast<std::uint32_t>(rng() % 40);
        std::vector<std::uint64_t> in_off(nm), out_off(nm), lens(nm), olens(nm), dl(nm);
        std::vector<std::uint8_t> rks(176ull * nm);
        std::uint64_t oi = 0, oo = 0;
        for (std::uint32_t i = 0; i < nm; ++i) {
          lens[i] = rng() % 9000;
          in_off[i] = oi;
          out_off[i] = oo;
          oi += (lens[i] + 15) / 16 * 16;
          oo += (lens[i] / 16 + 1) * 16;
          std::uint8_t kk[16];
          for (auto& x : kk) x = static_cast<std::uint8_t>(rng());
          paes_cuda_expand_key(kk, rks.data() + 176ull * i);
        }
        std::vector<std::uint8_t> src(oi + 16), enc(oo + 16), dec(oo + 16);
        fill(src, rng);
        EXPECT(paes_cuda_batch_host(0, src.data(), enc.data(), in_off.data(), out_off.data(), lens.data(), rks.data(),
                                    nm, 1, olens.data(), 0) == 0, "batch encrypt");
        EXPECT(paes_cuda_batch_host(1, enc.data(), dec.data(), out_off.data(), out_off.data(), olens.data(), rks.data(),
                                    nm, 1, dl.data(), 0) == 0, "batch decrypt");
        for (std::uint32_t i = 0; i < nm; ++i)
          EXPECT(dl[i] == lens[i] && std::memcmp(dec.data() + out_off[i], src.data() + in_off[i], lens[i]) == 0,
                 "batch round trip");
        break;
      }
      case 4: {  // file job round trip
        const std::string base = "/tmp/paes_stress_" + std::to_string(::getpid()) + "_" + std::to_string(id);
        {
          std::ofstream f(base + ".in", std::ios::binary);
          f.write(reinterpret_cast<const char*>(data.data()), static_cast<std::streamsize>(n));
        }
        paes_job_outcome o{};
        EXPECT(paes_cuda_run_job((base + ".in").c_str(), (base + ".enc").c_str(), key, 2, 0, &o) == 0, "file encrypt");
        // again over the existing output: the replaced file goes to the detached reclaim when it is large
        // enough (PAES_FILE_ASYNC_RECLAIM lowers the threshold in the sanitizer runs)
        EXPECT(paes_cuda_run_job((base + ".in").c_str(), (base + ".enc").c_str(), key, 1, 0, &o) == 0, "file re-encrypt");
        EXPECT(paes_cuda_run_job((base + ".enc").c_str(), (base + ".out").c_str(), key, 3, 1, &o) == 0, "file decrypt");
        std::ifstream g(base + ".out", std::ios::binary);
        std::vector<std::uint8_t> got((std::istreambuf_iterator<char>(g)), std::istreambuf_iterator<char>());
        EXPECT(got == data, "file round trip");
        for (const char* ext : {".in", ".enc", ".out"}) ::unlink((base + ext).c_str());
        break;
      }
      case 5: {  // single-state transforms
        std::vector<std::uint8_t> s(16 * 64), s2;
        fill(s, rng);
        s2 = s;
        EXPECT(paes_cuda_state_transform(PAES_OP_MIX_COLUMNS, s2.data(), 64, nullptr) == 0, "mix");
        EXPECT(paes_cuda_state_transform(PAES_OP_INV_MIX_COLUMNS, s2.data(), 64, nullptr) == 0, "inv mix");
        EXPECT(s2 == s, "state round trip");
        break;
      }
      default: {  // runtime reconfiguration under load
        if (rng() % 2) paes_cuda_set_zero_copy_max((rng() % 2) ? 0 : (128ull << 20));
        else paes_cuda_set_pipeline((rng() % 2) ? (8ull << 20) : (64ull << 20), 2 + static_cast<int>(rng() % 2));
        break;
      }
    }
  }
  cudaStreamDestroy(st);
}

int main(int argc, char** argv) {
  const int threads = argc > 1 ? std::atoi(argv[1]) : 8;
  const int iters = argc > 2 ? std::atoi(argv[2]) : 40;
  const int devs[4] = {0, 0, 0, 0};  // device 0 listed 4x: the multi-shard paths run on one GPU
  paes_cuda_set_devices(devs, 4);
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) pool.emplace_back(worker, t, iters);
  for (auto& t : pool) t.join();
  paes_cuda_set_pipeline(256ull << 20, 3);
  std::printf("stress: %d threads x %d ops, %d failures\n", threads, iters, g_fail.load());
  return g_fail.load();
}
