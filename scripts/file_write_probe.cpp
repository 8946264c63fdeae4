// How fast can a NEW tmpfs file of n bytes be filled from a host buffer?
// (run_job's output side, abi_file.cu.)  Page faults of a fresh shared mapping
// contend on the file's page-cache lock; this probe times the alternatives:
//   mmap_copy        T threads memcpy into a fresh MAP_SHARED mapping (the current writer)
//   mmap_copyK       the same with K < T threads
//   populateSM_copy  T threads madvise(MADV_POPULATE_WRITE) S MiB of the mapping at a time, then memcpy it
//   mmap_copy_after_falloc  one fallocate, then T threads memcpy through the mapping
//   pipe_falloc_mmapW  one allocator thread in 16 MiB steps, W writers copy 64 MiB pieces through the mapping behind it
//   turns_fallocSM_mmap  the same with S MiB steps, allocator and writers taking turns (never concurrent)
//   pwrite           T threads pwrite into the fresh file (pages allocated by write, not zeroed first)
//   falloc1+pwrite   one thread fallocates everything, then T threads pwrite
//   fallocK          K threads fallocate disjoint ranges (time only)
//   pipe_fallocK     K allocator threads run ahead in 64 MiB steps, T-K pwrite threads follow the watermark
// One JSON line.  No GPU needed.
//   g++ -O2 -std=c++20 -pthread scripts/file_write_probe.cpp -o scripts/file_write_probe_bin
//   scripts/file_write_probe_bin /dev/shm 4294967296 16
#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <shared_mutex>
#include <string>
#include <thread>
#include <vector>

static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

template <class F>
static void par(unsigned t, std::size_t n, F f) {
  std::vector<std::thread> pool;
  const std::size_t step = (((n + t - 1) / t) + 4095) & ~std::size_t(4095);
  for (unsigned i = 0; i < t; ++i) {
    const std::size_t b = std::min(n, i * step), e = std::min(n, (i + 1) * step);
    if (b < e) pool.emplace_back([=] { f(b, e - b); });
  }
  for (auto& th : pool) th.join();
}

static void pwrite_all(int fd, const char* p, std::size_t n, std::size_t off) {
  while (n) {
    const ssize_t r = ::pwrite(fd, p, std::min<std::size_t>(n, 8u << 20), static_cast<off_t>(off));
    if (r <= 0) { std::perror("pwrite"); std::exit(1); }
    p += r; off += r; n -= r;
  }
}

int main(int argc, char** argv) {
  const std::string dir = argc > 1 ? argv[1] : "/dev/shm";
  const std::size_t n = argc > 2 ? std::stoull(argv[2]) : (1ull << 30);
  const unsigned t = argc > 3 ? static_cast<unsigned>(std::stoul(argv[3])) : 16;
  const std::string out_path = dir + "/paes_wr_out";
  std::vector<char> src(n);
  par(t, n, [&](std::size_t b, std::size_t l) { std::memset(src.data() + b, 0x5a, l); });
  auto fresh = [&] {
    ::unlink(out_path.c_str());
    return ::open(out_path.c_str(), O_RDWR | O_CREAT | O_TRUNC, 0644);
  };
  std::printf("{\"bytes\": %zu, \"threads\": %u", n, t);
  for (int rep = 0; rep < 2; ++rep) {
    {
      const int fd = fresh();
      const double a = now();
      (void)!::ftruncate(fd, static_cast<off_t>(n));
      auto* p = static_cast<char*>(::mmap(nullptr, n, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0));
      par(t, n, [&](std::size_t b, std::size_t l) { std::memcpy(p + b, src.data() + b, l); });
      const double c = now();
      ::munmap(p, n);
      ::close(fd);
      std::printf(", \"mmap_copy_s_%d\": %.3f", rep, c - a);
    }
    for (unsigned tt : {t / 2, t / 4, t / 8}) {  // fewer faulting threads: is the fault path contended?
      if (!tt) continue;
      const int fd = fresh();
      const double a = now();
      (void)!::ftruncate(fd, static_cast<off_t>(n));
      auto* p = static_cast<char*>(::mmap(nullptr, n, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0));
      par(tt, n, [&](std::size_t b, std::size_t l) { std::memcpy(p + b, src.data() + b, l); });
      const double c = now();
      ::munmap(p, n);
      ::close(fd);
      std::printf(", \"mmap_copy%u_s_%d\": %.3f", tt, rep, c - a);
    }
    for (std::size_t step : {std::size_t(2) << 20, std::size_t(32) << 20}) {
      // each thread populates (allocate + zero + map, no per-page trap) a step of its range, then copies it
      const int fd = fresh();
      const double a = now();
      (void)!::ftruncate(fd, static_cast<off_t>(n));
      auto* p = static_cast<char*>(::mmap(nullptr, n, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0));
      par(t, n, [&](std::size_t b, std::size_t l) {
        for (std::size_t o = 0; o < l; o += step) {
          const std::size_t m = std::min(step, l - o);
          if (::madvise(p + b + o, m, 23 /* MADV_POPULATE_WRITE */) != 0) { std::perror("madvise"); }
          std::memcpy(p + b + o, src.data() + b + o, m);
        }
      });
      const double c = now();
      ::munmap(p, n);
      ::close(fd);
      std::printf(", \"populate%zuM_copy_s_%d\": %.3f", step >> 20, rep, c - a);
    }
    {
      // one fallocate (allocation only), then T threads copy through the mapping (faults zero + map)
      const int fd = fresh();
      const double a = now();
      (void)!::posix_fallocate(fd, 0, static_cast<off_t>(n));
      const double b0 = now();
      auto* p = static_cast<char*>(::mmap(nullptr, n, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0));
      par(t, n, [&](std::size_t b, std::size_t l) { std::memcpy(p + b, src.data() + b, l); });
      const double c = now();
      ::munmap(p, n);
      ::close(fd);
      std::printf(", \"mmap_copy_after_falloc_s_%d\": %.3f", rep, c - b0);
    }
    for (unsigned w : {t, t / 2, t / 4}) {
      // one allocator thread runs ahead in 16 MiB steps; W writers copy each 64 MiB piece through the mapping
      // once it is allocated (run_job's Prealloc, without the reads and the GPU)
      if (!w) continue;
      const int fd = fresh();
      constexpr std::size_t kStep = 16u << 20, kPiece = 64u << 20;
      std::atomic<std::size_t> mark{0};
      const double a = now();
      (void)!::ftruncate(fd, static_cast<off_t>(n));
      auto* p = static_cast<char*>(::mmap(nullptr, n, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0));
      double alloc_done = 0;
      std::thread alloc([&] {
        for (std::size_t o = 0; o < n; o += kStep) {
          (void)!::fallocate(fd, 0, static_cast<off_t>(o), static_cast<off_t>(std::min(kStep, n - o)));
          mark.store(std::min(n, o + kStep), std::memory_order_release);
        }
        alloc_done = now();
      });
      std::vector<std::thread> wr;
      for (unsigned i = 0; i < w; ++i)
        wr.emplace_back([&, i] {
          for (std::size_t b = 0; b < n; b += kPiece) {
            const std::size_t l = std::min(kPiece, n - b);
            while (mark.load(std::memory_order_acquire) < b + l) std::this_thread::yield();
            const std::size_t part = ((l + w - 1) / w + 4095) & ~std::size_t(4095);
            const std::size_t pb = std::min(l, i * part), pe = std::min(l, (i + 1) * part);
            if (pb < pe) std::memcpy(p + b + pb, src.data() + b + pb, pe - pb);
          }
        });
      alloc.join();
      for (auto& th : wr) th.join();
      const double c = now();
      ::munmap(p, n);
      ::close(fd);
      std::printf(", \"pipe_falloc_mmap%u_s_%d\": %.3f, \"pipe_falloc_mmap%u_alloc_done_s_%d\": %.3f", w, rep, c - a, w, rep,
                  alloc_done - a);
    }
    for (std::size_t kStep : {std::size_t(16) << 20, std::size_t(64) << 20, std::size_t(256) << 20}) {
      // the same, but allocator and writers never run at the same time: the allocator takes a lock exclusively per
      // step, the writers share it while they copy (faults and fallocate on one inode slow each other down)
      const unsigned w = t;
      const int fd = fresh();
      constexpr std::size_t kPiece = 64u << 20;
      std::atomic<std::size_t> mark{0};
      std::shared_mutex turn;
      const double a = now();
      (void)!::ftruncate(fd, static_cast<off_t>(n));
      auto* p = static_cast<char*>(::mmap(nullptr, n, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0));
      double alloc_done = 0;
      std::thread alloc([&] {
        for (std::size_t o = 0; o < n; o += kStep) {
          {
            std::unique_lock<std::shared_mutex> lk(turn);
            (void)!::fallocate(fd, 0, static_cast<off_t>(o), static_cast<off_t>(std::min(kStep, n - o)));
          }
          mark.store(std::min(n, o + kStep), std::memory_order_release);
        }
        alloc_done = now();
      });
      std::vector<std::thread> wr;
      for (unsigned i = 0; i < w; ++i)
        wr.emplace_back([&, i] {
          for (std::size_t b = 0; b < n; b += kPiece) {
            const std::size_t l = std::min(kPiece, n - b);
            while (mark.load(std::memory_order_acquire) < b + l) std::this_thread::yield();
            const std::size_t part = ((l + w - 1) / w + 4095) & ~std::size_t(4095);
            const std::size_t pb = std::min(l, i * part), pe = std::min(l, (i + 1) * part);
            if (pb < pe) {
              std::shared_lock<std::shared_mutex> lk(turn);
              std::memcpy(p + b + pb, src.data() + b + pb, pe - pb);
            }
          }
        });
      alloc.join();
      for (auto& th : wr) th.join();
      const double c = now();
      ::munmap(p, n);
      ::close(fd);
      std::printf(", \"turns_falloc%zuM_mmap_s_%d\": %.3f, \"turns_falloc%zuM_alloc_done_s_%d\": %.3f", kStep >> 20, rep, c - a,
                  kStep >> 20, rep, alloc_done - a);
    }
    for (unsigned tt : {t, t / 2, t / 4}) {
      const int fd = fresh();
      const double a = now();
      par(tt, n, [&](std::size_t b, std::size_t l) { pwrite_all(fd, src.data() + b, l, b); });
      const double c = now();
      ::close(fd);
      std::printf(", \"pwrite%u_s_%d\": %.3f", tt, rep, c - a);
    }
    {
      const int fd = fresh();
      const double a = now();
      (void)!::posix_fallocate(fd, 0, static_cast<off_t>(n));
      const double b0 = now();
      par(t, n, [&](std::size_t b, std::size_t l) { pwrite_all(fd, src.data() + b, l, b); });
      const double c = now();
      ::close(fd);
      std::printf(", \"falloc1_s_%d\": %.3f, \"pwrite_after_falloc_s_%d\": %.3f", rep, b0 - a, rep, c - b0);
    }
    for (unsigned k : {2u, 4u}) {
      const int fd = fresh();
      const double a = now();
      par(k, n, [&](std::size_t b, std::size_t l) { (void)!::posix_fallocate(fd, static_cast<off_t>(b), static_cast<off_t>(l)); });
      const double c = now();
      ::close(fd);
      std::printf(", \"falloc%u_s_%d\": %.3f", k, rep, c - a);
    }
    for (unsigned k : {1u, 2u}) {
      // K allocators run ahead in steps; the writers follow the lowest watermark
      const int fd = fresh();
      constexpr std::size_t kStep = 64u << 20;
      const std::size_t steps = (n + kStep - 1) / kStep;
      std::vector<std::atomic<unsigned char>> done(steps);
      for (auto& d : done) d.store(0);
      const double a = now();
      std::vector<std::thread> alloc;
      for (unsigned i = 0; i < k; ++i)
        alloc.emplace_back([&, i] {
          for (std::size_t s = i; s < steps; s += k) {
            const std::size_t b = s * kStep, l = std::min(kStep, n - b);
            (void)!::posix_fallocate(fd, static_cast<off_t>(b), static_cast<off_t>(l));
            done[s].store(1, std::memory_order_release);
          }
        });
      // writers: step s is split over the t-k writer threads
      const unsigned w = t - k;
      std::vector<std::thread> wr;
      for (unsigned i = 0; i < w; ++i)
        wr.emplace_back([&, i] {
          for (std::size_t s = 0; s < steps; ++s) {
            while (!done[s].load(std::memory_order_acquire)) std::this_thread::yield();
            const std::size_t b = s * kStep, l = std::min(kStep, n - b);
            const std::size_t part = ((l + w - 1) / w + 4095) & ~std::size_t(4095);
            const std::size_t pb = std::min(l, i * part), pe = std::min(l, (i + 1) * part);
            if (pb < pe) pwrite_all(fd, src.data() + b + pb, pe - pb, b + pb);
          }
        });
      for (auto& th : alloc) th.join();
      const double m = now();
      for (auto& th : wr) th.join();
      const double c = now();
      ::close(fd);
      std::printf(", \"pipe_falloc%u_s_%d\": %.3f, \"pipe_falloc%u_alloc_done_s_%d\": %.3f", k, rep, c - a, k, rep, m - a);
    }
  }
  std::printf("}\n");
  ::unlink(out_path.c_str());
  return 0;
}
