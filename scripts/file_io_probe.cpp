// Host-side limits of the file path (run_job on tmpfs): parallel pread into
// a buffer, and parallel copies into a fresh MAP_SHARED mapping of a new file
// -- as is (page faults allocate tmpfs pages), after fallocate, and after a
// parallel MADV_POPULATE_WRITE.  One JSON line.  No GPU needed.
//   g++ -O2 -std=c++20 -pthread scripts/file_io_probe.cpp -o /tmp/file_io_probe
//   /tmp/file_io_probe /dev/shm 4294967296 16
#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#ifndef MADV_POPULATE_WRITE
#define MADV_POPULATE_WRITE 23
#endif

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

int main(int argc, char** argv) {
  const std::string dir = argc > 1 ? argv[1] : "/dev/shm";
  const std::size_t n = argc > 2 ? std::stoull(argv[2]) : (1ull << 30);
  const unsigned t = argc > 3 ? static_cast<unsigned>(std::stoul(argv[3])) : 16;
  const std::string in_path = dir + "/paes_io_in", out_path = dir + "/paes_io_out";
  std::vector<char> src(n);
  par(t, n, [&](std::size_t b, std::size_t l) { std::memset(src.data() + b, 0x5a, l); });
  {
    const int fd = ::open(in_path.c_str(), O_RDWR | O_CREAT | O_TRUNC, 0644);
    par(t, n, [&](std::size_t b, std::size_t l) { (void)!::pwrite(fd, src.data() + b, l, static_cast<off_t>(b)); });
    ::close(fd);
  }
  std::printf("{\"bytes\": %zu, \"threads\": %u", n, t);
  // pread into an already-touched buffer
  {
    const int fd = ::open(in_path.c_str(), O_RDONLY);
    const double a = now();
    par(t, n, [&](std::size_t b, std::size_t l) { (void)!::pread(fd, src.data() + b, l, static_cast<off_t>(b)); });
    std::printf(", \"pread_gbs\": %.2f", n / (now() - a) / 1e9);
    ::close(fd);
  }
  auto map_copy = [&](int mode) {
    ::unlink(out_path.c_str());
    const int fd = ::open(out_path.c_str(), O_RDWR | O_CREAT | O_TRUNC, 0644);
    const double a = now();
    if (mode == 1) (void)!::posix_fallocate(fd, 0, static_cast<off_t>(n));
    else (void)!::ftruncate(fd, static_cast<off_t>(n));
    auto* p = static_cast<char*>(::mmap(nullptr, n, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0));
    const double b0 = now();
    if (mode == 2) par(t, n, [&](std::size_t b, std::size_t l) { ::madvise(p + b, l, MADV_POPULATE_WRITE); });
    const double b1 = now();
    par(t, n, [&](std::size_t b, std::size_t l) { std::memcpy(p + b, src.data() + b, l); });
    const double c = now();
    ::munmap(p, n);
    ::close(fd);
    return std::make_pair(n / (c - a) / 1e9, std::make_pair(b1 - b0 + (mode == 1 ? b0 - a : 0.0), c - b1));
  };
  const auto plain = map_copy(0);
  const auto falloc = map_copy(1);
  const auto popw = map_copy(2);
  std::printf(", \"mmap_copy_gbs\": %.2f, \"fallocate_then_copy_gbs\": %.2f, \"fallocate_s\": %.3f, \"copy_after_fallocate_s\": %.3f"
              ", \"populate_write_then_copy_gbs\": %.2f, \"populate_s\": %.3f, \"copy_after_populate_s\": %.3f}\n",
              plain.first, falloc.first, falloc.second.first, falloc.second.second, popw.first, popw.second.first,
              popw.second.second);
  ::unlink(in_path.c_str());
  ::unlink(out_path.c_str());
  return 0;
}
