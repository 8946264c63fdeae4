// Is pinning a pageable buffer on the fly cheap when it is backed by
// transparent huge pages?  scripts/host_register_probe.cu measured
// cudaHostRegister of 4 KiB-page malloc memory at 1-2 GB/s -- too slow to beat
// the staged ring.  The staged ring already advises MADV_HUGEPAGE on a
// pageable destination (runtime.cu advise_huge_pages); if registering such a
// range runs far above the ring's rate, the destination could be DMA'd into
// directly (no pinned output slot, no copy-out team).
// Rows per size: register / unregister GB/s for 4 KiB pages (touched), huge
// pages (touched), huge pages (fresh: the pin faults them in), the fault-in
// rate of fresh huge pages by memset, and AnonHugePages seen.  One JSON line.
// Build: scripts/build_probes.sh
#include <sys/mman.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <string>

#include <cuda_runtime.h>

#include "paes_cuda.h"

static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

static std::uint8_t* map(std::size_t n, bool huge) {
  void* p = mmap(nullptr, n, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  if (p == MAP_FAILED) return nullptr;
  madvise(p, n, huge ? MADV_HUGEPAGE : MADV_NOHUGEPAGE);
  return static_cast<std::uint8_t*>(p);
}

static long anon_huge_kb() {
  std::ifstream f("/proc/self/smaps_rollup");
  std::string k;
  long v;
  while (f >> k) {
    if (k == "AnonHugePages:") {
      f >> v;
      return v;
    }
  }
  return -1;
}

static std::string thp_mode() {
  std::ifstream f("/sys/kernel/mm/transparent_hugepage/enabled");
  std::string s;
  std::getline(f, s);
  return s;
}

int main() {
  cudaFree(nullptr);
  std::printf("{\"thp\": \"%s\", \"rows\": [", thp_mode().c_str());
  bool first = true;
  for (std::size_t n : {256ul << 20, 1ul << 30, 4ul << 30}) {
    double reg4k = 0, unreg4k = 0, reg_huge = 0, unreg_huge = 0, reg_fresh = 0, fault = 0;
    long huge_kb = 0;
    int ok = 1;
    const int reps = 3;
    for (int i = 0; i < reps; ++i) {
      // 4 KiB pages, touched
      std::uint8_t* a = map(n, false);
      std::memset(a, 1, n);
      double t = now();
      ok &= cudaHostRegister(a, n, cudaHostRegisterDefault) == cudaSuccess;
      reg4k += now() - t;
      t = now();
      ok &= cudaHostUnregister(a) == cudaSuccess;
      unreg4k += now() - t;
      munmap(a, n);
      // huge pages, touched (fault-in timed separately)
      std::uint8_t* b = map(n, true);
      t = now();
      std::memset(b, 1, n);
      fault += now() - t;
      huge_kb = anon_huge_kb();
      t = now();
      ok &= cudaHostRegister(b, n, cudaHostRegisterDefault) == cudaSuccess;
      reg_huge += now() - t;
      t = now();
      ok &= cudaHostUnregister(b) == cudaSuccess;
      unreg_huge += now() - t;
      munmap(b, n);
      // huge pages, fresh: the registration faults them in
      std::uint8_t* c = map(n, true);
      t = now();
      ok &= cudaHostRegister(c, n, cudaHostRegisterDefault) == cudaSuccess;
      reg_fresh += now() - t;
      ok &= cudaHostUnregister(c) == cudaSuccess;
      munmap(c, n);
    }
    auto gbs = [&](double s) { return reps * static_cast<double>(n) / s / 1e9; };
    std::printf("%s{\"bytes\": %zu, \"register_4k_gbs\": %.2f, \"unregister_4k_gbs\": %.2f, \"register_huge_gbs\": %.2f, "
                "\"unregister_huge_gbs\": %.2f, \"register_fresh_huge_gbs\": %.2f, \"memset_fault_huge_gbs\": %.2f, "
                "\"anon_huge_kb\": %ld, \"ok\": %d}",
                first ? "" : ", ", n, gbs(reg4k), gbs(unreg4k), gbs(reg_huge), gbs(unreg_huge), gbs(reg_fresh),
                gbs(fault), huge_kb, ok);
    first = false;
  }
  std::printf("], \"error\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
