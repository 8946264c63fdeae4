// gpu_worker.cpp -- a GPU worker that speaks the reference's hidden worker
// protocol.
//
//   paes_gpu_worker __worker --in P --offset N --len N --final 0|1
//                   --dir encrypt|decrypt --keyfd FD --out P [--device D]
//
// Same arguments, key-over-inherited-pipe convention and exit codes as the
// reference CLI's worker mode (paes_main.cpp:121-152 -> run_worker_chunk,
// exec.cpp:349-373), so the reference's UNMODIFIED process strategy
// (run_process_isolated, exec.cpp:272-338) drives B200s when its
// JobSpec::worker_exe points here: one process per chunk, one GPU each.
// The chunk goes through paes_cuda_worker_chunk: the library's pipelined
// file shard (parallel pread -> pinned ring -> kernel -> mapped output).
// Device: --device, else PAES_WORKER_DEVICE, else chunk i -> GPU i mod #GPUs.
// The protocol passes no chunk index, but the parent names chunk i's output
// "<output>.w<i>.<pid>.part" (exec.cpp:286-289), so i is read from --out.
// (The byte range alone does not determine i: shares differ by one block --
// 3,3,2,2 puts chunk 3 at offset / len = 4 -- and several worker counts can
// produce the same range at different indices.)  Only an --out of another
// shape falls back to offset / len.  --print-chunk-index prints i and exits
// (no key, no GPU), for tests.
//
// Exit codes (paes_main.cpp:316-325): 0 ok, 2 invalid argument, 1 anything else.
#include <unistd.h>

#include <algorithm>
#include <cctype>
#include <chrono>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "paes_cuda.h"

namespace {

int usage(const char* msg) {
  std::fprintf(stderr, "worker: %s\n", msg);
  return 2;
}

// i from the parent's "<output>.w<i>.<pid>.part" (exec.cpp:286-289), else offset / len.
std::uint64_t chunk_index(const std::string& out, std::uint64_t offset, std::uint64_t len) {
  const std::size_t w = out.rfind(".w");
  if (w != std::string::npos && out.size() > 5 && out.compare(out.size() - 5, 5, ".part") == 0) {
    std::size_t i = w + 2, j = i;
    while (j < out.size() && std::isdigit(static_cast<unsigned char>(out[j]))) ++j;
    std::size_t k = j + 1, m = k;
    while (m < out.size() && std::isdigit(static_cast<unsigned char>(out[m]))) ++m;
    if (j > i && j < out.size() && out[j] == '.' && m > k && out.compare(m, std::string::npos, ".part") == 0)
      return std::stoull(out.substr(i, j - i));
  }
  return len ? offset / len : 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2 || std::string(argv[1]) != "__worker") return usage("usage: paes_gpu_worker __worker --in ... --out ...");
  std::string in, out, dir;
  std::uint64_t offset = 0, len = 0;
  int final_flag = -1, keyfd = -1, device = -1;
  bool print_index = false;
  for (int i = 2; i < argc; i += 2) {
    const std::string k = argv[i];
    if (k == "--print-chunk-index") {
      print_index = true;
      --i;
      continue;
    }
    if (i + 1 >= argc) return usage(("missing value for " + k).c_str());
    const std::string v = argv[i + 1];
    try {
      if (k == "--in") in = v;
      else if (k == "--out") out = v;
      else if (k == "--dir") dir = v;
      else if (k == "--offset") offset = std::stoull(v);
      else if (k == "--len") len = std::stoull(v);
      else if (k == "--final") final_flag = std::stoi(v);
      else if (k == "--keyfd") keyfd = std::stoi(v);
      else if (k == "--device") device = std::stoi(v);
      else return usage(("unknown option " + k).c_str());
    } catch (const std::exception&) {
      return usage(("bad value for " + k).c_str());
    }
  }
  if (print_index && !out.empty()) {
    std::printf("%llu\n", static_cast<unsigned long long>(chunk_index(out, offset, len)));
    return 0;
  }
  if (in.empty() || out.empty() || final_flag < 0 || keyfd < 0) return usage("missing option");
  int d = -1;
  if (dir == "encrypt") d = PAES_ENCRYPT;
  else if (dir == "decrypt") d = PAES_DECRYPT;
  else return usage("bad --dir");

  std::uint8_t key[16];
  std::size_t got = 0;
  while (got < 16) {
    const ssize_t n = ::read(keyfd, key + got, 16 - got);
    if (n <= 0) break;
    got += static_cast<std::size_t>(n);
  }
  if (got != 16) {
    std::fprintf(stderr, "worker: could not read 16 key bytes from fd %d\n", keyfd);
    return 1;
  }
  if (keyfd != 0) ::close(keyfd);

  const auto t0 = std::chrono::steady_clock::now();
  const bool trace = std::getenv("PAES_WORKER_TRACE") != nullptr;
  auto mark = [&](const char* what) {
    if (trace)
      std::fprintf(stderr, "worker: %s at %.3f s\n", what,
                   std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
  };
  const int ndev = paes_cuda_device_count();
  mark("device count");
  if (ndev <= 0) {
    std::fprintf(stderr, "worker: no CUDA device\n");
    return 1;
  }
  if (device < 0 && std::getenv("PAES_WORKER_DEVICE")) device = std::atoi(std::getenv("PAES_WORKER_DEVICE"));
  if (device < 0) device = static_cast<int>(chunk_index(out, offset, len) % static_cast<std::uint64_t>(ndev));
  if (paes_cuda_set_devices(&device, 1) != PAES_OK) {
    std::fprintf(stderr, "worker: %s\n", paes_cuda_last_error());
    return 1;
  }

  mark("device selected");
  // a one-shot process: size the pinned ring to this chunk instead of the
  // library's 3 x 256 MiB default (pinning it dominated a short worker's life)
  const std::uint64_t slot = std::min<std::uint64_t>(64ull << 20, std::max<std::uint64_t>(4ull << 20, (len / 6 + 4095) & ~std::uint64_t(4095)));
  paes_cuda_set_pipeline(slot, 3);
  const int rc = paes_cuda_worker_chunk(in.c_str(), offset, len, final_flag, d, key, out.c_str(), device);
  mark("chunk done");
  const int code = rc == PAES_OK ? 0 : rc == PAES_EINVAL ? 2 : 1;
  if (rc != PAES_OK) std::fprintf(stderr, "worker: %s\n", paes_cuda_last_error());
  // The output file is complete and closed (paes_cuda_worker_chunk unmaps /
  // truncates it before returning).  Leave without the CUDA runtime's
  // teardown -- context destruction and unpinning took ~0.3 s of a short
  // worker's life; the kernel reclaims it all at exit anyway.
  std::fflush(nullptr);
  std::_Exit(code);
}
