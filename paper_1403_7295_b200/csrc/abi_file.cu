// abi_file.cu -- C ABI of the file path: run_job with the "gpu" strategy
// (exec.hpp:18-51, exec.cpp:340-347): parallel pread -> pinned ring -> H2D /
// kernel / D2H -> writer threads into a shared mapping of the temp file,
// rename on success (AtomicOutput, exec.cpp:80-106).
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <sys/vfs.h>
#include <unistd.h>

#include <cerrno>
#include <chrono>
#include <cstdio>
#include <sstream>
#include <thread>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "host_copy.hpp"
#include "runtime.hpp"

using namespace paes_b200;
using namespace paes_b200::rt;

// ============================================================ file path
namespace {

struct Fd {
  int fd = -1;
  ~Fd() {
    if (fd >= 0) ::close(fd);
  }
};

struct IoFail {
  std::string msg;
};

struct Map {
  std::uint8_t* p = nullptr;
  std::uint64_t n = 0;
  ~Map() {
    if (p) ::munmap(p, n);
  }
};

// The pages of a mapped output, allocated ahead of the writers.  A store to a
// fresh page of a shared tmpfs mapping allocates, zeroes and maps it inside the
// fault, and 8-16 threads faulting one file saturate at ~0.55 s per 4 GiB
// (scripts/file_write_probe.cpp: 1 thread 2.2 s, 4 threads 0.69, 8 0.53, 16
// 0.56).  fallocate(2) allocates the same pages without zeroing or mapping
// them at 0.30 s per 4 GiB from one thread (more threads serialise on the
// inode), and copies into already allocated pages then take 0.14-0.16 s with
// 16 threads.  So one thread runs fallocate over the shards' output regions in
// steps, round-robin, and each writer waits until the step holding its bytes is
// allocated: allocation overlaps the reads, the GPU and the copies instead of
// sitting inside every fault.  (Round 1 measured one fallocate of the whole
// file on a side thread with writers NOT waiting for it: slower, the faults
// and the allocator fought over the same pages.)  It also reserves the space:
// when the file system fills up, fallocate fails and the writers raise IoError
// instead of taking SIGBUS on a page that cannot be backed.
// PAES_FILE_PREALLOC=0 turns it off (writers fault the pages in themselves).
// Measured in the job (scripts/file_reclaim_ab.py --env PAES_FILE_PREALLOC,
// profiles/r02_file_prealloc_ab.json, 4 GiB on /dev/shm): 0.60-0.62 -> 0.52-0.55
// s.  The allocator is then the critical path and runs at ~0.5 s per 4 GiB, not
// its 0.30 s alone: the writers' faults on the same inode slow it.  Letting
// allocator and writers take turns on a shared_mutex, which in isolation gets
// the sum 0.30 + 0.16 s (file_write_probe turns_*), gave no gain in the job
// (0.60-0.61 s) and was dropped.
class Prealloc {
 public:
  struct Region {
    std::uint64_t off = 0, len = 0;
  };
  static constexpr std::uint64_t kStep = 16ull << 20;

  Prealloc() = default;
  Prealloc(const Prealloc&) = delete;
  Prealloc& operator=(const Prealloc&) = delete;
  ~Prealloc() { stop(); }

  void start(int fd, std::vector<Region> regions) {
    const char* e = std::getenv("PAES_FILE_PREALLOC");
    if ((e && e[0] == '0') || regions.empty()) return;
    fd_ = fd;
    regions_ = std::move(regions);
    done_.assign(regions_.size(), 0);
    active_ = true;
    th_ = std::thread([this] { run(); });
  }

  // Blocks until bytes [off, off + len) of the file are allocated; false when
  // the allocation failed (the caller reports the write failure).
  bool wait(std::uint64_t off, std::uint64_t len) {
    if (!active_ || !len) return true;
    std::size_t r = 0;
    while (r < regions_.size() && !(off >= regions_[r].off && off < regions_[r].off + regions_[r].len)) ++r;
    if (r == regions_.size()) return true;  // outside every region: nothing was promised
    const std::uint64_t need = std::min(off + len - regions_[r].off, regions_[r].len);
    const auto t0 = std::chrono::steady_clock::now();
    std::unique_lock<std::mutex> lk(mu_);
    cv_.wait(lk, [&] { return done_[r] >= need || failed_ || unsupported_; });
    waited_ns_ += std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count();
    return !failed_;
  }

  void stop() {
    if (!th_.joinable()) return;
    quit_.store(true, std::memory_order_relaxed);
    th_.join();
  }

 private:
  void run() {
    const auto t0 = std::chrono::steady_clock::now();
    struct Trace {
      std::chrono::steady_clock::time_point t0;
      Prealloc* self;
      ~Trace() {
        if (std::getenv("PAES_FILE_TRACE"))
          std::fprintf(stderr, "[paes file] prealloc thread ran %.3f s; writers waited %.3f s in total\n",
                       std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(),
                       self->waited_ns_.load() * 1e-9);
      }
    } trace{t0, this};
    std::vector<std::uint64_t> pos(regions_.size(), 0);
    for (bool more = true; more && !quit_.load(std::memory_order_relaxed);) {
      more = false;
      for (std::size_t r = 0; r < regions_.size() && !quit_.load(std::memory_order_relaxed); ++r) {
        if (pos[r] >= regions_[r].len) continue;
        const std::uint64_t n = std::min(kStep, regions_[r].len - pos[r]);
        int rc;
        do {
          rc = ::fallocate(fd_, 0, static_cast<off_t>(regions_[r].off + pos[r]), static_cast<off_t>(n));
        } while (rc != 0 && errno == EINTR);
        std::lock_guard<std::mutex> lk(mu_);
        if (rc != 0) {
          // no fallocate here: the writers allocate by faulting, as before;
          // anything else (ENOSPC, EDQUOT, EIO, EFBIG) fails the job
          if (errno == EOPNOTSUPP || errno == ENOSYS) unsupported_ = true;
          else failed_ = true;
          cv_.notify_all();
          return;
        }
        pos[r] += n;
        done_[r] = pos[r];
        cv_.notify_all();
        more = more || pos[r] < regions_[r].len;
      }
    }
  }

  int fd_ = -1;
  std::vector<Region> regions_;
  std::vector<std::uint64_t> done_;  // bytes allocated from each region's start (mu_)
  std::mutex mu_;
  std::condition_variable cv_;
  bool failed_ = false, unsupported_ = false;  // mu_
  bool active_ = false;
  std::atomic<bool> quit_{false};
  std::atomic<long long> waited_ns_{0};  // PAES_FILE_TRACE
  std::thread th_;
};

// Size the output to `cap` and pick the writer by file system.  On tmpfs
// (the paper's /dev/shm runs) the output is mapped shared and its pages are
// allocated by the writer threads' own faults, in parallel: preallocating with
// fallocate on a side thread was measured slower (scripts/ab_file_variants.py,
// profiles/r01_file_prealloc_ab.json).  On disk file systems plain pwrite
// from the pinned slots wins: 4 GiB on the box's ext4 root, 1.70 GB/s against
// 1.27 with the mapping (ext4's page_mkwrite per faulted page;
// profiles/r01_file_ext4_writer_ab.json).  File systems that refuse shared
// mmap take pwrite too.  PAES_FILE_WRITER=mmap|pwrite overrides the choice
// (tests exercise both); PAES_FILE_NO_MMAP=1 is the older spelling of pwrite.
void open_output(int fd, std::uint64_t cap, Map& map) {
  if (!cap || ::ftruncate(fd, static_cast<off_t>(cap)) != 0) return;
  bool use_map;
  const char* w = std::getenv("PAES_FILE_WRITER");
  const char* nm = std::getenv("PAES_FILE_NO_MMAP");
  if (w && std::strcmp(w, "mmap") == 0) {
    use_map = true;
  } else if ((w && std::strcmp(w, "pwrite") == 0) || (nm && nm[0] == '1')) {
    use_map = false;
  } else {
    struct statfs fs {};
    use_map = ::fstatfs(fd, &fs) == 0 && static_cast<unsigned long>(fs.f_type) == 0x01021994ul;  // TMPFS_MAGIC
  }
  if (!use_map) return;
  // A store to a page of a shared mapping that the file system cannot back
  // raises SIGBUS instead of returning ENOSPC, which would kill the process
  // and leave the .part file behind.  Map only when the free space covers
  // the whole output; otherwise pwrite, whose ENOSPC becomes IoError and the
  // temp file is removed (AtomicOutput, exec.cpp:80-106).  (Reserving with
  // fallocate instead was measured slower on tmpfs, see above.)
  // (PAES_FILE_SKIP_SPACE_CHECK=1 is a test hook: it lets the mapping through
  // on a file system that is too small, as if the space had been taken between
  // this check and the writes; the Prealloc thread's fallocate then fails and
  // the job reports IoError.)
  const char* skip = std::getenv("PAES_FILE_SKIP_SPACE_CHECK");
  struct statfs fs {};
  if (!(skip && skip[0] == '1') &&
      (::fstatfs(fd, &fs) != 0 ||
       static_cast<unsigned long long>(fs.f_bavail) * static_cast<unsigned long long>(fs.f_bsize) < cap))
    return;
  void* p = ::mmap(nullptr, cap, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  if (p != MAP_FAILED) {
    map.p = static_cast<std::uint8_t*>(p);
    map.n = cap;
  }
}

// A job that replaces an existing output frees that file's pages inside
// rename(2): 4 GiB of tmpfs pages cost ~0.2 s of the caller's time, a quarter
// of a warm 4 GiB job.  Holding a descriptor across the rename keeps the old
// inode alive, and closing it on a detached thread moves the freeing off the
// job's critical path; the directory entry is replaced atomically either way
// (AtomicOutput, exec.cpp:80-106).  Only worth a thread for large files;
// PAES_FILE_ASYNC_RECLAIM=0 turns it off.  A/B (scripts/file_reclaim_ab.py,
// profiles/r02_file_reclaim_ab.json): 4 GiB job 0.78 -> 0.59 s, and 5.2 -> 6.5
// GB/s by the wall clock of a back-to-back loop, which pays the reaper too.
struct ReplacedOutput {
  int fd = -1;
  explicit ReplacedOutput(const char* path) {
    // 0 = off, unset or 1 = files of at least 64 MiB, any other number = that
    // many bytes (the sanitizer stress lowers it to reach this path with small files)
    const char* e = std::getenv("PAES_FILE_ASYNC_RECLAIM");
    const unsigned long long v = e ? std::strtoull(e, nullptr, 10) : 1;
    if (v == 0) return;
    const long long min_size = v == 1 ? (64ll << 20) : static_cast<long long>(v);
    // only a plain file is ever opened (a FIFO would block in open, a device may have side effects)
    struct stat st {};
    if (::stat(path, &st) != 0 || !S_ISREG(st.st_mode) || st.st_size < min_size) return;
    fd = ::open(path, O_RDONLY | O_CLOEXEC | O_NONBLOCK | O_NOCTTY);
    if (fd >= 0 && (::fstat(fd, &st) != 0 || !S_ISREG(st.st_mode) || st.st_nlink != 1 || st.st_size < min_size)) {
      ::close(fd);
      fd = -1;
    }
  }
  // (Handing the job's own 4 GiB output mapping to the same thread for its
  // munmap was measured too: it only moved ~60 ms into the next job, whose
  // writer faults then contend with the unmapping -- job time 0.59 -> 0.65 s,
  // loop wall clock unchanged; profiles/r02_file_reclaim_ab.json.)
  void reclaim_later() {
    if (fd < 0) return;
    const int old = fd;
    fd = -1;
    try {
      std::thread([old] { ::close(old); }).detach();
    } catch (...) {
      ::close(old);
    }
  }
  ~ReplacedOutput() {
    if (fd >= 0) ::close(fd);
  }
};

void pread_all(int fd, std::uint8_t* p, std::uint64_t n, std::uint64_t off, const std::string& path) {
  std::uint64_t got = 0;
  while (got < n) {
    const ssize_t r = ::pread(fd, p + got, n - got, static_cast<off_t>(off + got));
    if (r < 0 && errno == EINTR) continue;
    if (r <= 0) throw IoFail{"short read: " + path};
    got += static_cast<std::uint64_t>(r);
  }
}

void pwrite_all(int fd, const std::uint8_t* p, std::uint64_t n, std::uint64_t off, const std::string& path) {
  std::uint64_t put = 0;
  while (put < n) {
    const ssize_t r = ::pwrite(fd, p + put, n - put, static_cast<off_t>(off + put));
    if (r < 0 && errno == EINTR) continue;
    if (r <= 0) throw IoFail{"write failed: " + path};
    put += static_cast<std::uint64_t>(r);
  }
}

// Split one pread/pwrite of a pinned slot across several host threads: a
// single thread copying from/to the page cache runs at a few GB/s, far below
// the PCIe rate the slot is DMA'd at.  Threads per shard = host threads /
// shards, at most 8.
unsigned g_io_threads_per_shard = 0;  // 0 = auto

template <class F>
void par_io(std::uint64_t n, unsigned threads, F&& f) {
  constexpr std::uint64_t kGrain = 4ull << 20;
  const std::uint64_t parts = std::min<std::uint64_t>(threads, (n + kGrain - 1) / kGrain);
  if (parts <= 1) {
    f(0, n);
    return;
  }
  const std::uint64_t step = (((n + parts - 1) / parts) + 4095) & ~std::uint64_t(4095);  // covers n
  std::vector<std::thread> pool;
  std::vector<std::string> errs(parts);
  for (std::uint64_t i = 1; i < parts; ++i) {
    const std::uint64_t b = std::min(n, i * step), e = std::min(n, (i + 1) * step);
    if (b >= e) break;
    pool.emplace_back([&, i, b, e] {
      try {
        f(b, e - b);
      } catch (const IoFail& x) {
        errs[i] = x.msg;
      }
    });
  }
  try {
    f(0, std::min(n, step));
  } catch (const IoFail& x) {
    errs[0] = x.msg;
  }
  for (auto& t : pool) t.join();
  for (const auto& e : errs)
    if (!e.empty()) throw IoFail{e};
}

// One GPU's shard of a file job: pread into pinned slots, H2D, kernel, D2H
// back into the same slot, pwrite -- all slots in flight at once.  Input
// bytes [in_off, in_off + r.in_len) land at out_off in the output (run_job:
// equal offsets; a worker chunk: its own file from 0).  Returns the output
// bytes written (decrypt final: unpadded).
std::uint64_t file_shard(DevCtx& d, const Range& r, int in_fd, int out_fd, std::uint8_t* out_map, Prealloc* pre,
                         std::uint64_t in_off, std::uint64_t out_off, const KeyWords& kw, const std::string& in_path,
                         const std::string& out_path, unsigned io_threads) {
  DeviceGuard g(d.id);
  {
    const auto t0 = std::chrono::steady_clock::now();
    ensure_pipeline(d, false);
    // pinned host slots sized to this job's piece, not to the device slot
    ensure_host_ring(d, piece_size(r.in_len, d.chunk, static_cast<int>(d.st.size())));  // slots carry 16 spare bytes for the pad block
    if (std::getenv("PAES_FILE_TRACE"))
      std::fprintf(stderr, "[paes file] rings ready in %.3f s (host slots %llu MiB)\n",
                   std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(),
                   static_cast<unsigned long long>(d.hbuf_bytes >> 20));
  }
  // on an exception, drain the slots' streams before d.mu is released: a
  // queued H2D may still read a pinned slot the next job would refill
  QuiesceOnThrow quiesce{d};
  const int S = static_cast<int>(d.st.size());
  const std::uint64_t C = piece_size(r.in_len, d.chunk, S);
  const std::uint64_t npieces = std::max<std::uint64_t>(1, (r.in_len + C - 1) / C);
  // Each slot's output is written back by its own writer thread (it waits on
  // the slot's event, then copies into the output mapping), so writing piece
  // k-1 overlaps reading piece k; a slot is refilled only after its writer
  // has been joined.
  std::vector<std::thread> writer(S);
  std::vector<std::string> werr(S);
  auto write_slot = [&](int s, std::uint64_t base, std::uint64_t len) {
    try {
      PAES_CK(cudaSetDevice(d.id));
      PAES_CK(cudaEventSynchronize(d.ev[s]));
      std::uint8_t* slot = d.hbuf[s];
      // both writers split the slot over the I/O threads: page faults of a
      // shared mapping proceed in parallel, and one pwrite per slot measured
      // slower on ext4 (1.22 vs 1.65 GB/s, 4 GiB)
      if (out_map) {
        // the piece's pages are allocated ahead by the job's Prealloc thread
        if (pre && !pre->wait(base, len)) throw IoFail{"write failed: " + out_path};
        par_io(len, io_threads, [&](std::uint64_t o, std::uint64_t n) { bulk_copy(out_map + base + o, slot + o, n); });
      } else
        par_io(len, io_threads, [&](std::uint64_t o, std::uint64_t n) { pwrite_all(out_fd, slot + o, n, base + o, out_path); });
    } catch (const IoFail& e) {
      werr[s] = e.msg;
    } catch (const CudaFail& e) {
      werr[s] = e.msg;
    }
  };
  auto join_slot = [&](int s) {
    if (writer[s].joinable()) writer[s].join();
    if (!werr[s].empty()) throw IoFail{werr[s]};
  };
  struct JoinAll {  // never leave a writer running on an exception
    std::vector<std::thread>& w;
    ~JoinAll() {
      for (auto& t : w)
        if (t.joinable()) t.join();
    }
  } join_all{writer};
  // the last piece's trailer check writes the mapped status word directly
  if (r.check_pad) *reinterpret_cast<volatile std::uint32_t*>(d.h_status) = 0xffffffffu;  // unchecked => PaddingError
  std::uint64_t out_total = 0;
  for (std::uint64_t k = 0; k < npieces; ++k) {
    const int s = static_cast<int>(k % S);
    join_slot(s);
    const std::uint64_t poff = k * C;
    const std::uint64_t len = std::min<std::uint64_t>(C, r.in_len - poff);
    const bool last = k + 1 == npieces;
    std::uint8_t* slot = d.hbuf[s];
    par_io(len, io_threads,
           [&](std::uint64_t o, std::uint64_t n) { pread_all(in_fd, slot + o, n, in_off + poff + o, in_path); });
    EcbArgs a = make_args(r, d.dbuf[s], d.dbuf[s], len, last, kw, d.m_status);
    if (len) PAES_CK(cudaMemcpyAsync(d.dbuf[s], d.hbuf[s], len, cudaMemcpyHostToDevice, d.st[s]));
    PAES_CK(launch_ecb(r.dec, a, d.sm_count, d.st[s]));
    const std::uint64_t olen = a.nblocks * 16;
    if (olen) PAES_CK(cudaMemcpyAsync(d.hbuf[s], d.dbuf[s], olen, cudaMemcpyDeviceToHost, d.st[s]));
    PAES_CK(cudaEventRecord(d.ev[s], d.st[s]));
    writer[s] = std::thread(write_slot, s, out_off + poff, olen);
    out_total = poff + olen;
  }
  for (int s = 0; s < S; ++s) join_slot(s);
  if (r.check_pad) {
    const std::uint32_t k = *reinterpret_cast<volatile std::uint32_t*>(d.h_status);
    if (k == 0xffffffffu) throw PaddingError("unpad: invalid pad bytes");
    out_total -= k;
  }
  return out_total;
}

}  // namespace

extern "C" int paes_cuda_run_job(const char* input_path, const char* output_path, const uint8_t key[16],
                                 uint32_t workers, int dir, paes_job_outcome* outcome) {
  const auto t0 = std::chrono::steady_clock::now();
  std::string tmp;
  const int rc = guarded([&] {
    if (!input_path || !output_path || !key) throw std::invalid_argument("null argument");
    if (dir != PAES_ENCRYPT && dir != PAES_DECRYPT) throw std::invalid_argument("bad dir");
    const bool dec = dir == PAES_DECRYPT;
    const std::string in_path(input_path), out_path(output_path);
    Fd in;
    in.fd = ::open(input_path, O_RDONLY);
    if (in.fd < 0) return fail(PAES_EIO, "cannot open input: " + in_path);
    struct stat stt {};
    if (::fstat(in.fd, &stt) != 0) return fail(PAES_EIO, "cannot stat input: " + in_path);
    const std::uint64_t len = static_cast<std::uint64_t>(stt.st_size);
    const auto devs = shard_devices(static_cast<int>(workers), len);
    const auto plan = dec ? plan_decrypt_chunks(len, static_cast<unsigned>(devs.size()))
                          : plan_chunks(len, static_cast<unsigned>(devs.size()));
    std::uint8_t rk[176];
    expand_key(key, rk);
    const KeyWords kw = dec ? dec_key_words(rk) : enc_key_words(rk);
    tmp = out_path + ".part." + std::to_string(::getpid());
    Fd out;
    out.fd = ::open(tmp.c_str(), O_RDWR | O_CREAT | O_TRUNC, 0644);
    if (out.fd < 0) return fail(PAES_EIO, "cannot open output: " + tmp);
    // Output through a shared mapping sized to the worst case (trimmed after
    // a decrypt's unpad); plain pwrite if the file system refuses mmap.
    const std::uint64_t cap = dec ? len : (len / 16 + 1) * 16;
    Map map;
    open_output(out.fd, cap, map);
    Prealloc pre;  // destroyed (joined) before the mapping and the descriptor go
    if (map.p) {
      std::vector<Prealloc::Region> regions;
      for (const Chunk& c : plan)
        regions.push_back({c.offset, dec ? c.raw_len : c.padded_len});
      pre.start(out.fd, std::move(regions));
    }
    std::vector<std::uint64_t> produced(plan.size(), 0);
    std::vector<std::string> failures(plan.size()), io_failures(plan.size());
    auto work = [&](std::size_t i) {
      const Chunk& c = plan[i];
      Range r;
      r.dec = dec;
      r.in_len = c.raw_len;
      r.pad = !dec && c.is_final;
      r.check_pad = dec && c.is_final;
      try {
        const auto td = std::chrono::steady_clock::now();
        DevCtx& d = device(devs[i]);
        if (std::getenv("PAES_FILE_TRACE"))
          std::fprintf(stderr, "[paes file] device context %.3f s (job clock at %.3f s)\n",
                       std::chrono::duration<double>(std::chrono::steady_clock::now() - td).count(),
                       std::chrono::duration<double>(td - t0).count());
        std::lock_guard<std::mutex> lk(d.mu);
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        const unsigned io = g_io_threads_per_shard
                                ? g_io_threads_per_shard
                                : std::clamp<unsigned>(hw / static_cast<unsigned>(plan.size()), 1u, 8u);
        produced[i] = file_shard(d, r, in.fd, out.fd, map.p, &pre, c.offset, c.offset, kw, in_path, tmp, io);
      } catch (const CudaFail& e) {
        failures[i] = e.msg;
      } catch (const IoFail& e) {
        io_failures[i] = e.msg;
      } catch (const std::exception& e) {
        failures[i] = e.what();
      }
    };
    if (plan.size() == 1) {
      work(0);
    } else {
      shard_pool().run(std::vector<int>(devs.begin(), devs.begin() + static_cast<std::ptrdiff_t>(plan.size())), work);
    }
    // reading or writing the files is the reference's IoError (read_file /
    // write_file, exec.cpp:48-76), whichever shard met it
    for (const auto& m : io_failures)
      if (!m.empty()) return fail(PAES_EIO, m);
    std::ostringstream failed;
    bool any = false;
    for (std::size_t i = 0; i < failures.size(); ++i) {
      if (failures[i].empty()) continue;
      failed << (any ? "; " : "") << "chunk " << i << ": " << failures[i];
      any = true;
    }
    if (any) return fail(PAES_EWORKER, "worker failure: " + failed.str());
    pre.stop();  // every region is allocated by now (each shard waited for its last piece)
    std::uint64_t total = 0;
    for (auto p : produced) total += p;
    if (::ftruncate(out.fd, static_cast<off_t>(total)) != 0) return fail(PAES_EIO, "truncate failed: " + tmp);
    {
      ReplacedOutput replaced(output_path);
      if (::rename(tmp.c_str(), output_path) != 0) return fail(PAES_EIO, "rename failed: " + out_path);
      replaced.reclaim_later();
    }
    tmp.clear();
    if (outcome) {
      outcome->bytes_in = len;
      outcome->bytes_out = total;
      outcome->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
    return PAES_OK;
  });
  if (rc != PAES_OK && !tmp.empty()) ::unlink(tmp.c_str());  // no partial output (exec.cpp:86-91)
  return rc;
}
// run_worker_chunk (exec.hpp:46-59, exec.cpp:349-373): one worker's chunk,
// file to file -- bytes [offset, offset + raw_len) of the input, padded or
// unpadded iff final, written to out_path from 0.  The same pipelined shard
// as run_job (pinned ring, parallel pread, writer threads into a mapping).
// Errors in the reference's order: IoError for the input first, then the
// chunk-transform rules (invalid_argument / PaddingError).
extern "C" int paes_cuda_worker_chunk(const char* input_path, uint64_t offset, uint64_t raw_len, int is_final,
                                      int dir, const uint8_t key[16], const char* output_path, int device) {
  return guarded([&] {
    try {
      if (!input_path || !output_path || !key) throw std::invalid_argument("null argument");
      if (dir != PAES_ENCRYPT && dir != PAES_DECRYPT) throw std::invalid_argument("bad dir");
      const std::string in_path(input_path), out_path(output_path);
      Fd in;
      in.fd = ::open(input_path, O_RDONLY);
      if (in.fd < 0) throw IoFail{"cannot open input: " + in_path};
      struct stat stt {};
      if (::fstat(in.fd, &stt) != 0) throw IoFail{"cannot stat input: " + in_path};
      const std::uint64_t size = static_cast<std::uint64_t>(stt.st_size);
      if (offset > size || raw_len > size - offset)
        throw IoFail{"short read of chunk [" + std::to_string(offset) + ", +" + std::to_string(raw_len) +
                     "): " + in_path};
      const bool dec = dir == PAES_DECRYPT;
      const bool final = is_final != 0;
      if (!final && raw_len % 16 != 0) throw std::invalid_argument("non-final chunk length must be a multiple of 16");
      if (dec && raw_len % 16 != 0) throw std::invalid_argument("decrypt: length must be a multiple of 16");
      if (dec && final && raw_len == 0) throw PaddingError("unpad: length must be a non-zero multiple of 16");
      Range r;
      r.dec = dec;
      r.in_len = raw_len;
      r.pad = !dec && final;
      r.check_pad = dec && final;
      std::uint8_t rk[176];
      expand_key(key, rk);
      const KeyWords kw = dec ? dec_key_words(rk) : enc_key_words(rk);
      const int dev = device >= 0 ? device : device_list(1)[0];
      Fd out;
      out.fd = ::open(output_path, O_RDWR | O_CREAT | O_TRUNC, 0644);
      if (out.fd < 0) throw IoFail{"cannot open output: " + out_path};
      const std::uint64_t cap = r.pad ? (raw_len / 16 + 1) * 16 : raw_len;
      Map map;
      open_output(out.fd, cap, map);
      Prealloc pre;
      if (map.p) pre.start(out.fd, {{0, cap}});
      std::uint64_t produced = 0;
      if (cap) {
        DevCtx& d = rt::device(dev);
        std::lock_guard<std::mutex> lk(d.mu);
        const unsigned io = g_io_threads_per_shard ? g_io_threads_per_shard
                                                   : std::clamp<unsigned>(std::thread::hardware_concurrency(), 1u, 8u);
        produced = file_shard(d, r, in.fd, out.fd, map.p, &pre, offset, 0, kw, in_path, out_path, io);
        pre.stop();
      }
      if (::ftruncate(out.fd, static_cast<off_t>(produced)) != 0) throw IoFail{"truncate failed: " + out_path};
      return PAES_OK;
    } catch (const IoFail& e) {
      return fail(PAES_EIO, e.msg);
    }
  });
}
