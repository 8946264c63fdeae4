// runtime.cu -- the host runtime behind the C ABI: per-device contexts, the
// multi-stream host<->device ring (zero-copy small path, pinned direct ring,
// staged ring for pageable memory) and the multi-GPU block-range sharder.
//
// Reference boundary: aes::encrypt_ecb/decrypt_ecb
// (aes.hpp:86-89), paes::encrypt_chunk/decrypt_chunk (exec.hpp:61-65) and
// run_job's strategy dispatch (exec.cpp:340-347).  Exceptions become codes:
// std::invalid_argument -> PAES_EINVAL, PaddingError -> PAES_EBADMSG,
// IoError -> PAES_EIO, WorkerError -> PAES_EWORKER, CUDA -> PAES_ECUDA.
#include <atomic>
#include <cuda_runtime.h>
#include <fcntl.h>
#include <pthread.h>
#include <sched.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cctype>
#include <cmath>
#include <cerrno>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <sstream>
#include <string>
#include <thread>
#include <vector>
#include "host_copy.hpp"
#include "runtime.hpp"

namespace paes_b200::rt {

thread_local std::string t_err;

int fail(int code, const std::string& msg) {
  t_err = msg;
  return code;
}


DevCtx g_dev[kMaxDev];
std::mutex g_cfg_mu;
std::vector<int> g_devices;  // empty = all visible
// Ring shape: 3 streams, slots of 256 MiB (piece_size() uses the full slot
// only for ranges beyond ~16 GiB; see there).
std::uint64_t g_chunk = 256ull << 20;
int g_streams = 3;
std::atomic<std::uint64_t> g_zero_copy_max{48ull << 20};  // scripts/ring_piece_sweep.py: the ring wins from ~64 MiB

// The device count is fixed for the life of a process once CUDA has
// initialised: cached after the first successful query (hot device-pointer
// calls validate their device index against it on every call).
int visible_devices() {
  static std::atomic<int> cached{-1};
  const int c = cached.load(std::memory_order_relaxed);
  if (c > 0) return c;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  if (n > 0) cached.store(n, std::memory_order_relaxed);
  return n;
}

void check_alias(const void* in, std::uint64_t in_len, const void* out, std::uint64_t out_len) {
  if (in == out || in_len == 0 || out_len == 0 || !in || !out) return;
  const std::uintptr_t a = reinterpret_cast<std::uintptr_t>(in), b = reinterpret_cast<std::uintptr_t>(out);
  if (a < b + out_len && b < a + in_len)
    throw std::invalid_argument("in and out overlap without being the same buffer (they may only alias exactly, "
                                "aes.hpp:84-85)");
}

// CPUs of a device's NUMA node (from sysfs via its PCI address); empty when
// the platform reports none.  Cached per device.
const cpu_set_t* device_numa_cpus(int dev) {
  static std::mutex mu;
  static cpu_set_t sets[kMaxDev];
  static int state[kMaxDev];  // 0 unknown, 1 have set, 2 none
  if (dev < 0 || dev >= kMaxDev) return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  if (state[dev] == 0) {
    state[dev] = 2;
    char bdf[32] = {0};
    if (cudaDeviceGetPCIBusId(bdf, sizeof bdf, dev) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    std::string id(bdf);
    for (auto& ch : id) ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch)));
    int node = -1;
    if (FILE* f = std::fopen(("/sys/bus/pci/devices/" + id + "/numa_node").c_str(), "r")) {
      if (std::fscanf(f, "%d", &node) != 1) node = -1;
      std::fclose(f);
    }
    if (node < 0) return nullptr;
    char list[4096] = {0};
    if (FILE* f = std::fopen(("/sys/devices/system/node/node" + std::to_string(node) + "/cpulist").c_str(), "r")) {
      if (!std::fgets(list, sizeof list, f)) list[0] = 0;
      std::fclose(f);
    }
    CPU_ZERO(&sets[dev]);
    int ncpu = 0;
    char* save = nullptr;
    for (char* tok = strtok_r(list, ",\n", &save); tok; tok = strtok_r(nullptr, ",\n", &save)) {
      int a = -1, b = -1;
      const int k = std::sscanf(tok, "%d-%d", &a, &b);
      if (k < 1) continue;
      if (k == 1) b = a;
      for (int c = a; c <= b && c < CPU_SETSIZE; ++c, ++ncpu) CPU_SET(c, &sets[dev]);
    }
    if (ncpu) state[dev] = 1;
  }
  return state[dev] == 1 ? &sets[dev] : nullptr;
}

void bind_thread_to_device_numa(int dev) {
  if (const cpu_set_t* s = device_numa_cpus(dev)) pthread_setaffinity_np(pthread_self(), sizeof(cpu_set_t), s);
}

// Lazily initialise a device: kernel attributes, status words.
DevCtx& device(int id) {
  const int n = visible_devices();
  if (id < 0 || id >= n || id >= kMaxDev)
    throw CudaFail{PAES_ENODEV, "no such CUDA device: " + std::to_string(id) + " (visible: " + std::to_string(n) + ")"};
  DevCtx& d = g_dev[id];
  if (d.ready.load(std::memory_order_acquire)) return d;
  std::lock_guard<std::mutex> lk(d.mu);
  if (!d.ready.load(std::memory_order_relaxed)) {
    DeviceGuard g(id);
    PAES_CK(cudaDeviceGetAttribute(&d.sm_count, cudaDevAttrMultiProcessorCount, id));
    PAES_CK(prepare_kernels());
    PAES_CK(cudaHostAlloc(reinterpret_cast<void**>(&d.h_status), 4096, cudaHostAllocMapped | cudaHostAllocPortable));
    PAES_CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d.m_status), d.h_status, 0));
    {
      std::lock_guard<std::mutex> sl(d.slot_mu);
      d.free_slots.clear();
      for (int i = 1024 - 1; i >= 1; --i) d.free_slots.push_back(i);  // 4096 B = 1024 words; word 0 is d.mu's
    }
    PAES_CK(cudaMalloc(&d.d_acc, 64));
    PAES_CK(cudaMallocHost(&d.h_acc, 64));
    d.id = id;
    d.ready.store(true, std::memory_order_release);
  }
  return d;
}

StatusSlot::StatusSlot(DevCtx& d) : d_(d) {
  {
    std::lock_guard<std::mutex> lk(d.slot_mu);
    if (!d.free_slots.empty()) {
      idx_ = d.free_slots.back();
      d.free_slots.pop_back();
      return;
    }
  }
  fallback_ = std::unique_lock<std::mutex>(d.mu);  // all slots busy: word 0, serialised
}

StatusSlot::~StatusSlot() {
  if (idx_ != 0) {
    std::lock_guard<std::mutex> lk(d_.slot_mu);
    d_.free_slots.push_back(idx_);
  }
}

// Pipeline buffers (device rings + optional pinned host ring); d.mu held.
void ensure_pipeline(DevCtx& d, bool need_host) {
  std::uint64_t chunk;
  int ns;
  {
    std::lock_guard<std::mutex> lk(g_cfg_mu);
    chunk = g_chunk;
    ns = g_streams;
  }
  auto release = [&d] {
    for (auto s : d.st) cudaStreamSynchronize(s);
    for (auto p : d.dbuf) cudaFree(p);
    for (auto p : d.hbuf) cudaFreeHost(p);
    for (auto p : d.sin_buf) cudaFreeHost(p);
    for (auto p : d.sout_buf) cudaFreeHost(p);
    for (auto p : d.obuf) cudaFree(p);
    for (auto p : d.dsc) cudaFree(p);
    for (auto s : d.st) cudaStreamDestroy(s);
    for (auto e : d.ev) cudaEventDestroy(e);
    for (auto* v : {&d.ev_in, &d.ev_k, &d.ev_out}) {
      for (auto e : *v) cudaEventDestroy(e);
      v->clear();
    }
    d.dbuf.clear();
    d.hbuf.clear();
    d.hbuf_bytes = 0;
    d.sin_buf.clear();
    d.sout_buf.clear();
    d.obuf.clear();
    d.dsc.clear();
    d.dsc_cap.clear();
    d.st.clear();
    d.ev.clear();
    d.chunk = 0;  // unconfigured: the next call builds the ring afresh
  };
  // A failed allocation (e.g. a pipeline too large for the device) must not
  // leave a half-built ring that later calls would index: everything is
  // released and the context is marked unconfigured before the error leaves.
  if (d.chunk != chunk || static_cast<int>(d.st.size()) != ns || static_cast<int>(d.dbuf.size()) != ns) {
    release();
    try {
      for (int i = 0; i < ns; ++i) {
        cudaStream_t s;
        PAES_CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        d.st.push_back(s);
        for (auto* v : {&d.ev, &d.ev_in, &d.ev_k, &d.ev_out}) {
          cudaEvent_t e;
          PAES_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
          v->push_back(e);
        }
        std::uint8_t* p = nullptr;
        PAES_CK(cudaMalloc(&p, chunk + 16));
        d.dbuf.push_back(p);
      }
    } catch (...) {
      release();
      throw;
    }
    d.chunk = chunk;
  }
  if (need_host) ensure_host_ring(d, d.chunk);
}

// Pinning is the expensive part of building the rings (3 x 256 MiB of
// cudaMallocHost cost ~0.3 s of a fresh process's first file job,
// scripts/file_cold_probe.py), and file pieces are at most 64 MiB up to 16 GiB
// of input (piece_size), so the host slots follow the job's piece.
void ensure_host_ring(DevCtx& d, std::uint64_t bytes) {
  const std::size_t ns = d.st.size();
  std::uint64_t want = 16ull << 20;
  while (want < bytes) want <<= 1;
  want = std::min<std::uint64_t>(want, std::max<std::uint64_t>(d.chunk, bytes));
  if (d.hbuf.size() == ns && d.hbuf_bytes >= want) return;
  for (auto p : d.hbuf) cudaFreeHost(p);
  d.hbuf.clear();
  d.hbuf_bytes = 0;
  try {
    for (std::size_t i = 0; i < ns; ++i) {
      std::uint8_t* p = nullptr;
      PAES_CK(cudaMallocHost(&p, want + 16));
      d.hbuf.push_back(p);
    }
  } catch (...) {
    for (auto p : d.hbuf) cudaFreeHost(p);
    d.hbuf.clear();
    throw;
  }
  d.hbuf_bytes = want;
}

std::vector<int> device_list(int ngpus) {
  std::vector<int> list;
  {
    std::lock_guard<std::mutex> lk(g_cfg_mu);
    list = g_devices;
  }
  if (list.empty()) {
    const int n = visible_devices();
    for (int i = 0; i < n; ++i) list.push_back(i);
  }
  if (list.empty()) throw CudaFail{PAES_ENODEV, "no CUDA device visible"};
  if (ngpus < 0) throw std::invalid_argument("ngpus must be >= 0");
  if (ngpus > 0) {
    if (ngpus > static_cast<int>(list.size()))
      throw CudaFail{PAES_ENODEV, "requested " + std::to_string(ngpus) + " GPUs, " + std::to_string(list.size()) +
                                      " available"};
    list.resize(ngpus);
  }
  return list;
}

std::vector<int> shard_devices(int ngpus, std::uint64_t len) {
  std::vector<int> devs = device_list(ngpus);
  if (ngpus == 0) devs.resize(auto_shards(len, static_cast<unsigned>(devs.size())));
  return devs;
}

void ShardPool::loop(Worker* w) {
  int bound = -1;
  for (;;) {
    std::function<void()> job;
    int dev;
    {
      std::unique_lock<std::mutex> lk(w->mu);
      w->cv.wait(lk, [w] { return static_cast<bool>(w->job); });
      job = std::move(w->job);
      w->job = nullptr;
      dev = w->dev;
    }
    if (dev != bound) {
      bind_thread_to_device_numa(dev);
      bound = dev;
    }
    try {
      job();
    } catch (...) {  // callers wrap their work in guarded(); never let a pool thread die
    }
    {
      std::lock_guard<std::mutex> lk(done_mu_);
      if (--pending_ == 0) done_cv_.notify_all();
    }
  }
}

void ShardPool::run(const std::vector<int>& devs, const std::function<void(std::size_t)>& f) {
  std::lock_guard<std::mutex> call(call_mu_);
  while (workers_.size() < devs.size()) {
    workers_.push_back(std::make_unique<Worker>());
    Worker* w = workers_.back().get();
    w->th = std::thread([this, w] { loop(w); });
  }
  {
    std::lock_guard<std::mutex> lk(done_mu_);
    pending_ = devs.size();
  }
  for (std::size_t k = 0; k < devs.size(); ++k) {
    Worker& w = *workers_[k];
    std::lock_guard<std::mutex> lk(w.mu);
    w.dev = devs[k];
    w.job = [&f, k] { f(k); };
    w.cv.notify_one();
  }
  std::unique_lock<std::mutex> lk(done_mu_);
  done_cv_.wait(lk, [this] { return pending_ == 0; });
}

ShardPool& shard_pool() {
  static ShardPool* pool = new ShardPool();  // leaked on purpose: parked threads outlive static destructors
  return *pool;
}

EcbArgs make_args(const Range& r, const std::uint8_t* in, std::uint8_t* out, std::uint64_t in_len, bool last,
                  const KeyWords& kw, std::uint32_t* status) {
  EcbArgs a{};
  a.in = in;
  a.out = out;
  a.nfull = in_len / 16;
  a.tail_len = static_cast<std::uint32_t>(in_len % 16);
  a.nblocks = a.nfull + ((r.pad && last) ? 1 : 0);
  a.check_pad = (r.check_pad && last) ? 1u : 0u;
  a.status = status;
  a.k = kw;
  return a;
}

// Piece size of the file path (abi_file.cu) and the host batch groups
// (abi_batch.cu), from measurements on the box (scripts/e2e_ring_sweep.py,
// pcie_probe.py, batch_host_probe.py); the pinned and staged rings have their
// own (pinned_piece_size, staged_piece_size):
// - short ranges: ~2 pieces per stream so copy-in, kernel and copy-out overlap;
// - up to ~16 GiB: 64 MiB pieces (1 GiB: 46.1 GB/s at 64 MiB against 44.6 at
//   both 33 MB and 128 MiB);
// - beyond: len / 256, up to the ring slot (64 GiB in place: 49.3 GB/s at
//   256 MiB against 48.3 at 64 MiB -- fewer per-piece gaps).
std::uint64_t piece_size(std::uint64_t len, std::uint64_t chunk, int streams) {
  constexpr std::uint64_t kMid = 64ull << 20;
  const std::uint64_t floor_piece = std::min<std::uint64_t>(4ull << 20, chunk);
  std::uint64_t p = len / (2ull * static_cast<std::uint64_t>(streams));
  if (p > kMid) p = std::max(kMid, len / 256);
  p = (p + 15) & ~std::uint64_t(15);
  return std::clamp(p, floor_piece, chunk);
}

// Piece size of the pinned direct ring (separate copy-in / kernel / copy-out
// queues, run_host_range): ~16 pieces while they stay >= 8 MiB, at most
// 64 MiB up to ~16 GiB, then len / 256 up to the slot.  Measured on 1x B200
// (scripts/ring_piece_sweep.py, profiles/r01_ring_piece_sweep.jsonl): 256 MiB
// 43.7 GB/s at 16 MiB pieces against 41.9 at the old len/6; 1 and 4 GiB best
// at 32-64 MiB (46.2 / 47.8); pieces below 8 MiB lose ~19 us each.
std::uint64_t pinned_piece_size(std::uint64_t len, std::uint64_t chunk) {
  constexpr std::uint64_t kMin = 8ull << 20, kMid = 64ull << 20, kBig = 16ull << 30;
  std::uint64_t p = len > kBig ? std::max(kMid, len / 256) : std::clamp(len / 16, kMin, kMid);
  p = (p + 15) & ~std::uint64_t(15);
  return std::clamp<std::uint64_t>(p, 16, chunk);
}

// Piece lengths of the pinned ring over `len` bytes with nominal piece C.
// The first copy-in and the last copy-out of a range run with nothing to
// overlap them, so the ring ramps: C/8, C/4, C/2, C, ..., C, C/2, C/4, C/8
// (every piece a multiple of 16 except the last, which takes the tail).
// PAES_RING_RAMP=0 gives flat C pieces (A/B).
std::vector<std::uint64_t> ring_pieces(std::uint64_t len, std::uint64_t C) {
  static const bool ramp = [] {
    const char* e = std::getenv("PAES_RING_RAMP");
    return !(e && e[0] == '0');
  }();
  std::vector<std::uint64_t> p;
  const std::uint64_t r1 = (C / 8) & ~std::uint64_t(15), r2 = (C / 4) & ~std::uint64_t(15),
                      r3 = (C / 2) & ~std::uint64_t(15);
  const std::uint64_t ramps = 2 * (r1 + r2 + r3);
  if (!ramp || r1 == 0 || len < ramps + 2 * C) {
    for (std::uint64_t off = 0; off < len || p.empty(); off += C) p.push_back(std::min(C, len - off));
    return p;
  }
  p = {r1, r2, r3};
  std::uint64_t mid = len - ramps;  // >= 2C
  const std::uint64_t q = mid / C;
  for (std::uint64_t i = 0; i < q; ++i) p.push_back(C);
  mid -= q * C;
  if (mid & ~std::uint64_t(15)) p.push_back(mid & ~std::uint64_t(15));
  p.insert(p.end(), {r3, r2, r1 + (mid & 15)});
  return p;
}

// What a host-pointer entry was handed.  Page-locked host memory (under UVA
// every cudaHostAlloc'd or registered buffer is device-accessible) carries
// its device alias; pageable and managed memory are copied by the host; a
// device pointer is the caller's mistake (the device-pointer entries take
// those) and is rejected before the host could dereference it.
struct HostPtr {
  const std::uint8_t* alias = nullptr;  // device alias of the buffer's start, or nullptr
  std::uint8_t* at(std::uint64_t off) const {
    return alias ? const_cast<std::uint8_t*>(alias) + off : nullptr;
  }
};

HostPtr classify_host(const void* p, const char* what) {
  HostPtr h;
  if (!p) return h;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return h;
  }
  if (a.type == cudaMemoryTypeDevice)
    throw std::invalid_argument(std::string(what) + " is device memory: host-pointer entries take host buffers "
                                "(use the *_device entry points for device buffers)");
  if (a.type == cudaMemoryTypeHost) h.alias = static_cast<const std::uint8_t*>(a.devicePointer);
  return h;
}

// ------------------------------------------------------------ short calls
// Short host ranges run as ONE kernel that reads and writes host memory over
// PCIe (zero-copy) -- no device ring, no copy-engine commands:
// - pinned caller buffers up to g_zero_copy_max: the kernel works on the
//   caller's buffers through their UVA aliases.  Measured against the copy
//   ring (profiles/r01_zero_copy_probe.json): 3.4x at 1 MiB, ahead up to
//   ~256 MiB; beyond that the copy engines' larger PCIe requests win (46 vs
//   40 GB/s at 1 GiB);
// - pageable buffers up to kBounceMax: pieces of kBouncePiece copied into
//   one of two mapped pinned bounce buffers, the kernel in place on it, copied
//   out -- double-buffered, so piece k's kernel runs while the host copies
//   piece k-1 out and piece k+1 in (replaces H2D + launch + D2H, three
//   commands and their latencies, and the staged ring's two copy teams and
//   drainer, whose fixed cost is ~300 us: encrypt_bytes of 1 MiB + 7 took
//   300-420 us there, 512 KiB 77 us here; profiles/r02_pageable_small_ab.txt).
// Each call leases a LANE of the device -- a stream, a mapped status word and
// (after the first pageable call) a bounce buffer of its own -- from a pool,
// instead of taking d.mu: short calls from many host threads overlap their
// launch, kernel and synchronisation latencies rather than queueing behind
// one lock (scripts/concurrent_small_probe.cu).  Lanes are created on demand,
// reused, and never freed; the pool holds as many as the peak number of
// concurrent short calls, at most kMaxLanes (a stream + 4 KiB mapped, + 1 MiB
// pinned once used for pageable data, per lane).
constexpr std::uint64_t kBouncePiece = 512ull << 10;  // a multiple of 16
constexpr std::uint64_t kBounceMax = 4ull << 20;

struct Lane {
  cudaStream_t st = nullptr;
  std::uint32_t* status_host = nullptr;  // mapped pinned page: word 0 trailer status, word 16 completion flag
  std::uint32_t* status_dev = nullptr;
  unsigned* ctr = nullptr;  // device word: CTAs of the lane's current kernel that have finished (EcbArgs::done_ctr)
  unsigned seq = 0;         // last completion value handed to a kernel
  std::uint8_t* bounce_host = nullptr;  // mapped pinned, 2 x (kBouncePiece + 16), lazy
  std::uint8_t* bounce_dev = nullptr;
  cudaEvent_t done[2] = {nullptr, nullptr};  // kernel on bounce half 0 / 1 finished
};

struct LanePool {
  std::mutex mu;
  std::condition_variable cv;
  std::vector<Lane*> free;
  int created = 0;
};
LanePool g_lanes[kMaxDev];
// Lanes per device: beyond this many concurrent short calls, callers wait for
// a lane (bounds the pool at 64 streams and 64 MiB of pinned bounce buffers;
// the 16-thread probe uses 16).
constexpr int kMaxLanes = 64;

class LaneLease {
 public:
  explicit LaneLease(DevCtx& d) : pool_(g_lanes[d.id]) {
    {
      std::unique_lock<std::mutex> lk(pool_.mu);
      pool_.cv.wait(lk, [this] { return !pool_.free.empty() || pool_.created < kMaxLanes; });
      if (!pool_.free.empty()) {
        lane_ = pool_.free.back();
        pool_.free.pop_back();
        return;
      }
      ++pool_.created;  // reserved; released again if the lane cannot be built
    }
    auto* l = new Lane();
    try {
      PAES_CK(cudaStreamCreateWithFlags(&l->st, cudaStreamNonBlocking));
      void* p = nullptr;
      PAES_CK(cudaHostAlloc(&p, 4096, cudaHostAllocMapped | cudaHostAllocPortable));
      l->status_host = static_cast<std::uint32_t*>(p);
      PAES_CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&l->status_dev), p, 0));
      l->status_host[16] = 0;
      PAES_CK(cudaMalloc(reinterpret_cast<void**>(&l->ctr), sizeof(unsigned)));
      PAES_CK(cudaMemset(l->ctr, 0, sizeof(unsigned)));
    } catch (...) {
      if (l->ctr) cudaFree(l->ctr);
      if (l->status_host) cudaFreeHost(l->status_host);
      if (l->st) cudaStreamDestroy(l->st);
      delete l;
      {
        std::lock_guard<std::mutex> lk(pool_.mu);
        --pool_.created;
      }
      pool_.cv.notify_one();
      throw;
    }
    lane_ = l;
  }
  ~LaneLease() {
    // a call that failed with work queued drains it before the lane is reused
    if (std::uncaught_exceptions() > depth_) cudaStreamSynchronize(lane_->st);
    {
      std::lock_guard<std::mutex> lk(pool_.mu);
      pool_.free.push_back(lane_);
    }
    pool_.cv.notify_one();
  }
  LaneLease(const LaneLease&) = delete;
  LaneLease& operator=(const LaneLease&) = delete;
  Lane& operator*() const { return *lane_; }

 private:
  LanePool& pool_;
  Lane* lane_ = nullptr;
  int depth_ = std::uncaught_exceptions();
};

// CTAs of a zero-copy launch.  Its rate is set by PCIe, not the SMs (32 SMs
// cipher ~190 GB/s), and fewer CTAs issuing host reads overlap reads with
// writes better: 4 MiB pinned 29.0 -> 34.1 GB/s, 16 MiB 36.6 -> 38.3, 48 MiB
// 38.9 -> 39.5, 1 MiB 22.4 -> 23.8 against one CTA per SM (both pools of
// runs in profiles/r02_zero_copy_grid_ab.txt).  It also leaves the other SMs
// to concurrent calls on other lanes.  PAES_ZC_GRID overrides it (A/B).
int zero_copy_grid(int sm_count) {
  static const int g = [] {
    const char* e = std::getenv("PAES_ZC_GRID");
    const int v = e ? std::atoi(e) : 0;
    return v > 0 ? v : 32;
  }();
  return std::min(g, sm_count);
}

// One zero-copy launch on the lane's stream over host memory (device aliases
// din/dout), synchronised; returns the bytes written.  A checked trailer's
// verdict lands in the lane's mapped word (finish_check reads it).
// Completion of a lane's kernels.  The kernel's last CTA writes a sequence
// number into the lane's mapped page after fencing every thread's writes to
// system scope (EcbArgs::done_flag); the host spins on that word instead of
// synchronising the stream, which skips the grid-completion semaphore round
// trip: launch + completion of a one-CTA kernel 12.6 -> 9.3 us, 32 CTAs 16.0
// -> 12.6-13.2 (scripts/sync_latency_probe.cu, profiles/r02_sync_latency.json).
// The spin polls the stream every 1024 rounds, so a failed kernel surfaces its
// error instead of hanging.  PAES_LANE_FLAG=0 synchronises the stream (A/B).
bool lane_flags_on() {
  static const bool on = [] {
    const char* e = std::getenv("PAES_LANE_FLAG");
    return !(e && e[0] == '0');
  }();
  return on;
}

void arm_completion(Lane& l, EcbArgs& a) {
  if (!lane_flags_on()) return;
  a.done_ctr = l.ctr;
  a.done_flag = l.status_dev + 16;
  a.done_seq = ++l.seq;
}

// Waits until the lane's kernel that carries `seq` has finished (its writes
// are visible to the host); earlier kernels on the lane finished before it.
void wait_completion(Lane& l, unsigned seq) {
  if (!lane_flags_on()) {
    PAES_CK(cudaStreamSynchronize(l.st));
    return;
  }
  const volatile unsigned* flag = l.status_host + 16;
  for (unsigned spin = 1;; ++spin) {
    if (static_cast<int>(*flag - seq) >= 0) break;
    if ((spin & 1023) == 0) {
      const cudaError_t e = cudaStreamQuery(l.st);
      if (e == cudaErrorNotReady) continue;
      if (e != cudaSuccess) {
        cudaGetLastError();
        throw CudaFail{PAES_ECUDA, std::string("lane kernel: ") + cudaGetErrorString(e)};
      }
      if (static_cast<int>(*flag - seq) >= 0) break;  // finished: the flag is visible now
      throw CudaFail{PAES_ECUDA, "lane kernel finished without its completion flag"};
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);  // host reads of the output after the flag
}

std::uint64_t lane_launch(DevCtx& d, Lane& l, const Range& r, const void* din, void* dout, const KeyWords& kw) {
  if (r.check_pad) *reinterpret_cast<volatile std::uint32_t*>(l.status_host) = 0xffffffffu;  // unchecked => PaddingError
  EcbArgs a = make_args(r, static_cast<const std::uint8_t*>(din), static_cast<std::uint8_t*>(dout), r.in_len, true,
                        kw, l.status_dev);
  arm_completion(l, a);
  PAES_CK(launch_ecb(r.dec, a, zero_copy_grid(d.sm_count), l.st));
  wait_completion(l, a.done_seq);
  return a.nblocks * 16;
}

// Output length after the trailer check (decrypt, final): unpadded, or PaddingError.
std::uint64_t finish_check(const Lane& l, const Range& r, std::uint64_t olen) {
  if (!r.check_pad) return olen;
  const std::uint32_t k = *reinterpret_cast<volatile std::uint32_t*>(l.status_host);
  if (k == 0xffffffffu) throw PaddingError("unpad: invalid pad bytes");
  return olen - k;
}

std::uint64_t configured_chunk() {
  std::lock_guard<std::mutex> lk(g_cfg_mu);
  return g_chunk;
}

// Pageable range through the lane's two bounce halves (see above).  Piece k's
// kernel is queued before the host copies piece k-1 out, so kernel and host
// copies overlap; half k%2 is refilled only after piece k-2 was copied out.
// Every output block is copied out (decrypt_ecb writes the whole span), then
// a checked trailer is settled.
std::uint64_t run_bounce(DevCtx& d, Lane& l, const Range& r, const std::uint8_t* in, std::uint8_t* out,
                         const KeyWords& kw) {
  constexpr std::uint64_t kHalf = kBouncePiece + 16;
  if (!l.bounce_host) {  // all or nothing: a half-built bounce must not be reused
    void* p = nullptr;
    std::uint8_t* dp = nullptr;
    cudaEvent_t ev[2] = {nullptr, nullptr};
    try {
      PAES_CK(cudaHostAlloc(&p, 2 * kHalf, cudaHostAllocMapped | cudaHostAllocPortable));
      PAES_CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dp), p, 0));
      for (auto& e : ev) PAES_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    } catch (...) {
      for (auto e : ev)
        if (e) cudaEventDestroy(e);
      if (p) cudaFreeHost(p);
      throw;
    }
    l.bounce_host = static_cast<std::uint8_t*>(p);
    l.bounce_dev = dp;
    l.done[0] = ev[0];
    l.done[1] = ev[1];
  }
  if (r.check_pad) *reinterpret_cast<volatile std::uint32_t*>(l.status_host) = 0xffffffffu;  // unchecked => PaddingError
  // balanced pieces of at most kBouncePiece (a 7-byte tail must not become a
  // piece of its own with nothing to overlap)
  const std::uint64_t want = std::max<std::uint64_t>(1, (r.in_len + kBouncePiece - 1) / kBouncePiece);
  const std::uint64_t C =
      std::clamp<std::uint64_t>(((r.in_len + want - 1) / want + 15) & ~std::uint64_t(15), 16, kBouncePiece);
  const std::uint64_t npieces = std::max<std::uint64_t>(1, (r.in_len + C - 1) / C);
  const int grid = zero_copy_grid(d.sm_count);
  std::uint64_t prev_off = 0, prev_len = 0, total = 0;
  unsigned prev_seq = 0;
  for (std::uint64_t k = 0; k < npieces; ++k) {
    const int h = static_cast<int>(k & 1);
    const std::uint64_t off = k * C;
    const std::uint64_t len = std::min(C, r.in_len - off);
    if (len) std::memcpy(l.bounce_host + h * kHalf, in + off, len);
    EcbArgs a = make_args(r, l.bounce_dev + h * kHalf, l.bounce_dev + h * kHalf, len, k + 1 == npieces, kw,
                          l.status_dev);
    arm_completion(l, a);
    PAES_CK(launch_ecb(r.dec, a, grid, l.st));
    if (!lane_flags_on()) PAES_CK(cudaEventRecord(l.done[h], l.st));
    if (k) {  // piece k-1, while piece k's kernel runs
      if (lane_flags_on()) wait_completion(l, prev_seq);
      else PAES_CK(cudaEventSynchronize(l.done[h ^ 1]));
      std::memcpy(out + prev_off, l.bounce_host + (h ^ 1) * kHalf, prev_len);
    }
    prev_off = off;
    prev_len = a.nblocks * 16;
    prev_seq = a.done_seq;
    total = off + prev_len;
  }
  if (lane_flags_on()) wait_completion(l, prev_seq);
  else PAES_CK(cudaEventSynchronize(l.done[(npieces - 1) & 1]));
  if (prev_len) std::memcpy(out + prev_off, l.bounce_host + ((npieces - 1) & 1) * kHalf, prev_len);
  return finish_check(l, r, total);
}

// The short-call path for this range, if it has one (no d.mu; see above).
// Returns false when the range belongs to a ring.
bool run_short(DevCtx& d, const Range& r, const std::uint8_t* in, std::uint8_t* out, const void* din, void* dout,
               const KeyWords& kw, std::uint64_t* produced) {
  const bool zero_copy = din && dout && r.in_len && r.in_len <= g_zero_copy_max.load(std::memory_order_relaxed);
  if (!zero_copy && r.in_len > std::min(kBounceMax, configured_chunk())) return false;
  DeviceGuard g(d.id);
  LaneLease lease(d);
  Lane& l = *lease;
  if (zero_copy) {
    *produced = finish_check(l, r, lane_launch(d, l, r, din, dout, kw));
    return true;
  }
  *produced = run_bounce(d, l, r, in, out, kw);
  return true;
}

cudaError_t copy_h2d_aligned(void* dev, const void* host, std::uint64_t n, cudaStream_t s) {
  const std::uint64_t head = (4096 - reinterpret_cast<std::uintptr_t>(host) % 4096) % 4096;
  if (head == 0 || head >= n) return cudaMemcpyAsync(dev, host, n, cudaMemcpyHostToDevice, s);
  const cudaError_t e = cudaMemcpyAsync(dev, host, head, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return e;
  return cudaMemcpyAsync(static_cast<std::uint8_t*>(dev) + head, static_cast<const std::uint8_t*>(host) + head, n - head,
                         cudaMemcpyHostToDevice, s);
}

cudaError_t copy_d2h_aligned(void* host, const void* dev, std::uint64_t n, cudaStream_t s) {
  const std::uint64_t head = (4096 - reinterpret_cast<std::uintptr_t>(host) % 4096) % 4096;
  if (head == 0 || head >= n) return cudaMemcpyAsync(host, dev, n, cudaMemcpyDeviceToHost, s);
  const cudaError_t e = cudaMemcpyAsync(host, dev, head, cudaMemcpyDeviceToHost, s);
  if (e != cudaSuccess) return e;
  return cudaMemcpyAsync(static_cast<std::uint8_t*>(host) + head, static_cast<const std::uint8_t*>(dev) + head, n - head,
                         cudaMemcpyDeviceToHost, s);
}

CopyTeam::CopyTeam(unsigned threads, int dev) {
  for (unsigned i = 1; i < std::max(1u, threads); ++i) th_.emplace_back([this, i, dev] { worker(i, dev); });
}

CopyTeam::~CopyTeam() {
  {
    std::lock_guard<std::mutex> lk(mu_);
    stop_ = true;
  }
  go_.notify_all();
  for (auto& t : th_) t.join();
}

void CopyTeam::worker(unsigned idx, int dev) {
  bind_thread_to_device_numa(dev);
  std::uint64_t seen = 0;
  for (;;) {
    std::uint8_t* dst;
    const std::uint8_t* src;
    std::uint64_t b, e;
    {
      std::unique_lock<std::mutex> lk(mu_);
      go_.wait(lk, [&] { return stop_ || gen_ != seen; });
      if (stop_) return;
      seen = gen_;
      dst = dst_;
      src = src_;
      b = std::min(n_, idx * step_);
      e = std::min(n_, (idx + 1) * step_);
    }
    if (b < e) bulk_copy(dst + b, src + b, e - b);
    {
      std::lock_guard<std::mutex> lk(mu_);
      if (--pending_ == 0) done_.notify_all();
    }
  }
}

void CopyTeam::copy(std::uint8_t* dst, const std::uint8_t* src, std::uint64_t n) {
  if (n == 0) return;
  const std::uint64_t parts = th_.size() + 1;
  if (parts == 1 || n < (1ull << 20)) {
    std::memcpy(dst, src, n);
    return;
  }
  std::lock_guard<std::mutex> call(call_mu_);
  const std::uint64_t step = (((n + parts - 1) / parts) + 4095) & ~std::uint64_t(4095);  // covers n
  {
    std::lock_guard<std::mutex> lk(mu_);
    dst_ = dst;
    src_ = src;
    n_ = n;
    step_ = step;
    pending_ = static_cast<unsigned>(th_.size());
    ++gen_;
  }
  go_.notify_all();
  bulk_copy(dst, src, std::min(n, step));
  std::unique_lock<std::mutex> lk(mu_);
  done_.wait(lk, [&] { return pending_ == 0; });
}

// Pageable host buffers (std::vector, Python bytes): the driver's own staging
// of pageable cudaMemcpyAsync serialises at ~7 GB/s, so the library stages
// through pinned slots itself.  Two host copy teams work at once: the calling
// thread's team copies piece k into an input slot while a drainer thread's
// team copies finished pieces out of the output slots, and the device side
// runs the pinned ring's three queues in between (copy-in stream, kernel
// stream, copy-out stream).  Piece k's device copy-out into output slot s
// waits until the drainer has emptied it (piece k-S).  Before: one thread did
// copy-out then copy-in per piece with a fresh thread team each time
// (1 GiB 18.1 GB/s, 64 MiB 8.7).
constexpr std::uint64_t kStagedSlot = 64ull << 20;

#ifndef PAES_STAGED_DIV
#define PAES_STAGED_DIV 8
#endif
#ifndef PAES_STAGED_MIN_KIB
#define PAES_STAGED_MIN_KIB 4096
#endif
std::uint64_t staged_piece_size(std::uint64_t len, std::uint64_t chunk) {
  const std::uint64_t p =
      std::clamp<std::uint64_t>(len / PAES_STAGED_DIV, std::uint64_t(PAES_STAGED_MIN_KIB) << 10, kStagedSlot);
  return std::min((p + 15) & ~std::uint64_t(15), chunk);  // chunk: the device slot (a multiple of 16)
}

void ensure_staged(DevCtx& d) {
  const std::size_t S = d.st.size();
  if (d.sin_buf.size() != S || d.sout_buf.size() != S) {
    auto free_all = [&d] {
      for (auto p : d.sin_buf) cudaFreeHost(p);
      for (auto p : d.sout_buf) cudaFreeHost(p);
      d.sin_buf.clear();
      d.sout_buf.clear();
    };
    free_all();
    try {
      for (std::size_t i = 0; i < S; ++i) {
        std::uint8_t* p = nullptr;
        PAES_CK(cudaMallocHost(&p, kStagedSlot + 16));
        d.sin_buf.push_back(p);
        p = nullptr;
        PAES_CK(cudaMallocHost(&p, kStagedSlot + 16));
        d.sout_buf.push_back(p);
      }
    } catch (...) {
      free_all();
      throw;
    }
  }
  if (!d.team_in) {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const unsigned t = std::clamp(hw / 2, 1u, 8u);  // two teams share the node's cores
    d.team_in = std::make_unique<CopyTeam>(t, d.id);
    d.team_out = std::make_unique<CopyTeam>(t, d.id);
  }
}

// A pageable destination is often fresh memory (a new bytes object or
// std::vector): every 4 KiB page faults in as the copy-out team first writes
// it, and the faults, not the ring, then bound the call (4 GiB encrypt_bytes
// 9.1 GB/s against 20.3 into pre-faulted memory,
// profiles/r02_pageable_probe.jsonl).  Asking for transparent huge pages on
// the 2 MiB-aligned part of the range (THP "madvise" mode, the usual default)
// makes those faults 512x fewer.  Only whole huge pages inside [out, out+n),
// which the call overwrites entirely, are advised.
void advise_huge_pages(std::uint8_t* out, std::uint64_t n) {
  constexpr std::uintptr_t kHuge = 2ull << 20;
  if (n < 4 * kHuge) return;
  const std::uintptr_t b = (reinterpret_cast<std::uintptr_t>(out) + kHuge - 1) & ~(kHuge - 1);
  const std::uintptr_t e = (reinterpret_cast<std::uintptr_t>(out) + n) & ~(kHuge - 1);
  if (e > b) (void)::madvise(reinterpret_cast<void*>(b), e - b, MADV_HUGEPAGE);  // advisory: errors ignored
}

std::uint64_t run_host_range_staged(DevCtx& d, const Range& r, const std::uint8_t* in, std::uint8_t* out,
                                    const KeyWords& kw) {
  ensure_pipeline(d, false);
  ensure_staged(d);
  advise_huge_pages(out, r.pad ? (r.in_len / 16 + 1) * 16 : r.in_len);
  QuiesceOnThrow quiesce{d};
  const int S = static_cast<int>(d.st.size());
  const std::uint64_t C = staged_piece_size(r.in_len, d.chunk);
  const std::uint64_t npieces = std::max<std::uint64_t>(1, (r.in_len + C - 1) / C);
  cudaStream_t sin = d.st[0], sk = d.st[1 % S], sout = d.st[2 % S];
  // the last piece's trailer check writes the mapped status word directly
  if (r.check_pad) *reinterpret_cast<volatile std::uint32_t*>(d.h_status) = 0xffffffffu;  // unchecked => PaddingError
  std::vector<std::uint64_t> olens(npieces, 0);
  std::mutex mu;
  std::condition_variable cv;
  std::uint64_t enqueued = 0, drained = 0;  // pieces whose copy-out is queued / copied to `out`
  bool abort = false;
  std::string drain_err;
  std::thread drainer([&] {
    cudaSetDevice(d.id);
    bind_thread_to_device_numa(d.id);
    for (std::uint64_t j = 0; j < npieces; ++j) {
      {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return enqueued > j || abort; });
        if (abort) return;
      }
      const cudaError_t e = cudaEventSynchronize(d.ev_out[j % S]);
      if (e != cudaSuccess) {
        std::lock_guard<std::mutex> lk(mu);
        drain_err = std::string("cudaEventSynchronize: ") + cudaGetErrorString(e);
        abort = true;
        cv.notify_all();
        return;
      }
      d.team_out->copy(out + j * C, d.sout_buf[j % S], olens[j]);
      {
        std::lock_guard<std::mutex> lk(mu);
        drained = j + 1;
      }
      cv.notify_all();
    }
  });
  auto stop_drainer = [&] {
    {
      std::lock_guard<std::mutex> lk(mu);
      abort = true;
    }
    cv.notify_all();
    drainer.join();
  };
  try {
    for (std::uint64_t k = 0; k < npieces; ++k) {
      const int s = static_cast<int>(k % S);
      const std::uint64_t off = k * C;
      const std::uint64_t len = std::min<std::uint64_t>(C, r.in_len - off);
      const bool last = k + 1 == npieces;
      const bool reuse = k >= static_cast<std::uint64_t>(S);
      if (reuse) PAES_CK(cudaEventSynchronize(d.ev_in[s]));  // input slot read by piece k-S's copy-in
      d.team_in->copy(d.sin_buf[s], in + off, len);
      EcbArgs a = make_args(r, d.dbuf[s], d.dbuf[s], len, last, kw, d.m_status);
      olens[k] = a.nblocks * 16;
      if (reuse) PAES_CK(cudaStreamWaitEvent(sin, d.ev_out[s], 0));  // device slot read by piece k-S's copy-out
      if (len) PAES_CK(cudaMemcpyAsync(d.dbuf[s], d.sin_buf[s], len, cudaMemcpyHostToDevice, sin));
      PAES_CK(cudaEventRecord(d.ev_in[s], sin));
      PAES_CK(cudaStreamWaitEvent(sk, d.ev_in[s], 0));
      PAES_CK(launch_ecb(r.dec, a, d.sm_count, sk));
      PAES_CK(cudaEventRecord(d.ev_k[s], sk));
      if (reuse) {  // output slot emptied by the drainer (piece k-S)
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return drained >= k - S + 1 || abort; });
        if (abort) break;
      }
      PAES_CK(cudaStreamWaitEvent(sout, d.ev_k[s], 0));
      if (olens[k]) PAES_CK(cudaMemcpyAsync(d.sout_buf[s], d.dbuf[s], olens[k], cudaMemcpyDeviceToHost, sout));
      PAES_CK(cudaEventRecord(d.ev_out[s], sout));
      {
        std::lock_guard<std::mutex> lk(mu);
        enqueued = k + 1;
      }
      cv.notify_all();
    }
  } catch (...) {
    stop_drainer();
    throw;
  }
  drainer.join();
  if (!drain_err.empty()) throw CudaFail{PAES_ECUDA, drain_err};
  for (auto st : d.st) PAES_CK(cudaStreamSynchronize(st));
  std::uint64_t out_total = (npieces - 1) * C + olens[npieces - 1];
  if (r.check_pad) {
    const std::uint32_t k = *reinterpret_cast<volatile std::uint32_t*>(d.h_status);
    if (k == 0xffffffffu) throw PaddingError("unpad: invalid pad bytes");
    out_total -= k;
  }
  return out_total;
}

// Host range on one device beyond the short-call path (d.mu held): pageable
// -> staged ring; pinned (both buffers) -> direct ring.  Returns the number of
// output bytes (decrypt with trailer check: unpadded).
std::uint64_t run_host_range(DevCtx& d, const Range& r, const std::uint8_t* in, std::uint8_t* out, bool pinned,
                             const KeyWords& kw) {
  DeviceGuard g(d.id);
  ensure_pipeline(d, false);
  if (!pinned) return run_host_range_staged(d, r, in, out, kw);
  QuiesceOnThrow quiesce{d};
  const int S = static_cast<int>(d.st.size());
  const std::vector<std::uint64_t> pieces = ring_pieces(r.in_len, pinned_piece_size(r.in_len, d.chunk));
  const std::uint64_t npieces = pieces.size();
  // the last piece's trailer check writes the mapped status word directly
  if (r.check_pad) *reinterpret_cast<volatile std::uint32_t*>(d.h_status) = 0xffffffffu;  // unchecked => PaddingError
  // One queue per engine: copy-in on st[0], kernels on st[1], copy-out on
  // st[2] (roles wrap with fewer streams), events between them per slot.
  // Piece k+S's copy-in waits only for piece k's copy-out (its slot), so the
  // copy-in engine runs ahead and copy-out always has a piece queued; with
  // all three steps of a piece on one stream, each kernel sat between its two
  // copies and its launch/completion latency stalled the copy engines
  // (scripts/ring_overhead_probe.cu, 1 GiB, empty kernel: 43.3 -> 45.0 GB/s at
  // 8 MiB pieces, 46.2 -> 47.1 at 16 MiB).
  cudaStream_t sin = d.st[0], sk = d.st[1 % S], sout = d.st[2 % S];
  std::uint64_t out_total = 0, off = 0;
  for (std::uint64_t k = 0; k < npieces; off += pieces[k], ++k) {
    const int s = static_cast<int>(k % S);
    const std::uint64_t len = pieces[k];
    const bool last = k + 1 == npieces;
    EcbArgs a = make_args(r, d.dbuf[s], d.dbuf[s], len, last, kw, d.m_status);
    if (k >= static_cast<std::uint64_t>(S)) PAES_CK(cudaStreamWaitEvent(sin, d.ev_out[s], 0));
    if (len) PAES_CK(copy_h2d_aligned(d.dbuf[s], in + off, len, sin));
    PAES_CK(cudaEventRecord(d.ev_in[s], sin));
    PAES_CK(cudaStreamWaitEvent(sk, d.ev_in[s], 0));
    PAES_CK(launch_ecb(r.dec, a, d.sm_count, sk));
    PAES_CK(cudaEventRecord(d.ev_k[s], sk));
    PAES_CK(cudaStreamWaitEvent(sout, d.ev_k[s], 0));
    const std::uint64_t olen = a.nblocks * 16;
    if (olen) PAES_CK(copy_d2h_aligned(out + off, d.dbuf[s], olen, sout));
    PAES_CK(cudaEventRecord(d.ev_out[s], sout));
    out_total = off + olen;
  }
  for (auto s : d.st) PAES_CK(cudaStreamSynchronize(s));
  if (r.check_pad) {
    const std::uint32_t k = *reinterpret_cast<volatile std::uint32_t*>(d.h_status);
    if (k == 0xffffffffu) throw PaddingError("unpad: invalid pad bytes");
    out_total -= k;
  }
  return out_total;
}

// Shard a host buffer over devices with the plan_chunks rule (encrypt) or
// plan_decrypt_chunks (decrypt); output offsets equal input offsets.
int host_transform(int dir, const std::uint8_t* in, std::uint64_t len, bool is_final, const std::uint8_t* rk,
                   std::uint8_t* out, std::uint64_t* out_len, int ngpus) {
  if (dir != PAES_ENCRYPT && dir != PAES_DECRYPT) throw std::invalid_argument("dir must be 0 (encrypt) or 1 (decrypt)");
  if (!rk) throw std::invalid_argument("null round keys");
  const bool dec = dir == PAES_DECRYPT;
  if (!is_final && len % 16 != 0) throw std::invalid_argument("non-final chunk length must be a multiple of 16");
  if (dec && len % 16 != 0) throw std::invalid_argument("decrypt: length must be a multiple of 16");
  if (len && !in) throw std::invalid_argument("null input");
  if (dec && is_final && len == 0) throw PaddingError("unpad: length must be a non-zero multiple of 16");
  if (len == 0 && !(is_final && !dec)) {
    if (out_len) *out_len = 0;
    return PAES_OK;
  }
  if (!out) throw std::invalid_argument("null output");
  check_alias(in, len, out, (is_final && !dec) ? (len / 16 + 1) * 16 : len);
  const HostPtr hin = classify_host(in, "input"), hout = classify_host(out, "output");
  const auto devs = shard_devices(ngpus, len);
  const KeyWords kw = dec ? dec_key_words(rk) : enc_key_words(rk);
  const auto plan = dec ? plan_decrypt_chunks(len, static_cast<unsigned>(devs.size()))
                        : plan_chunks(len, static_cast<unsigned>(devs.size()));
  std::vector<std::uint64_t> produced(plan.size(), 0);
  std::vector<int> codes(plan.size(), PAES_OK);
  std::vector<std::string> msgs(plan.size());
  auto work = [&](std::size_t i) {
    const Chunk& c = plan[i];
    Range r;
    r.dec = dec;
    r.in_len = c.raw_len;
    r.pad = !dec && is_final && c.is_final;
    r.check_pad = dec && is_final && c.is_final;
    codes[i] = guarded([&] {
      DevCtx& d = device(devs[i]);
      if (run_short(d, r, in + c.offset, out + c.offset, hin.at(c.offset), hout.at(c.offset), kw, &produced[i]))
        return PAES_OK;  // no d.mu
      std::lock_guard<std::mutex> lk(d.mu);
      produced[i] = run_host_range(d, r, in + c.offset, out + c.offset, hin.alias && hout.alias, kw);
      return PAES_OK;
    });
    if (codes[i]) msgs[i] = t_err;
  };
  if (plan.size() == 1) {
    work(0);
  } else {  // one persistent library thread per shard, on its GPU's NUMA node
    shard_pool().run(std::vector<int>(devs.begin(), devs.begin() + static_cast<std::ptrdiff_t>(plan.size())), work);
  }
  for (std::size_t i = 0; i < plan.size(); ++i)
    if (codes[i]) return fail(codes[i], msgs[i]);
  std::uint64_t total = 0;
  for (auto p : produced) total += p;
  if (out_len) *out_len = total;
  return PAES_OK;
}


void set_device_list(const std::vector<int>& ids) {
  std::lock_guard<std::mutex> lk(g_cfg_mu);
  g_devices = ids;
}

void set_zero_copy_max(std::uint64_t bytes) { g_zero_copy_max.store(bytes, std::memory_order_relaxed); }

void set_pipeline_config(std::uint64_t chunk_bytes, int streams) {
  std::lock_guard<std::mutex> lk(g_cfg_mu);
  if (chunk_bytes) g_chunk = chunk_bytes;
  if (streams) g_streams = streams;
}

}  // namespace paes_b200::rt
