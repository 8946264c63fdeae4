// runtime.hpp -- internal runtime shared by the C-ABI translation units:
// error mapping (C++ exceptions -> PAES_* codes), per-device contexts, the
// device list / pipeline configuration and the host<->device stream ring.
// Not installed; the public boundary is include/paes_cuda.h.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <exception>
#include <functional>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/paes_cuda.h"
#include "host_rules.hpp"
#include "launch.hpp"

namespace paes_b200::rt {

extern thread_local std::string t_err;
int fail(int code, const std::string& msg);

struct CudaFail {
  int code;
  std::string msg;
};

// A failed call's error is also left in the runtime's per-thread "last
// error" (non-sticky errors such as cudaErrorMemoryAllocation); it is
// cleared here, so a later launch check (cudaGetLastError) does not report it
// again after the caller has recovered.
#define PAES_CK(call)                                                                           \
  do {                                                                                          \
    const cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess) {                                                                    \
      cudaGetLastError();                                                                       \
      throw CudaFail{PAES_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)};            \
    }                                                                                           \
  } while (0)

// Runs `f`, mapping C++ exceptions to C-ABI codes (no exception crosses the ABI).
template <class F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const CudaFail& e) {
    return fail(e.code, e.msg);
  } catch (const PaddingError& e) {
    return fail(PAES_EBADMSG, e.what());
  } catch (const std::invalid_argument& e) {
    return fail(PAES_EINVAL, e.what());
  } catch (const std::bad_alloc&) {
    return fail(PAES_ECUDA, "host allocation failed");
  } catch (const std::exception& e) {
    return fail(PAES_ECUDA, e.what());
  }
}

class DeviceGuard {
 public:
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev_) != cudaSuccess) prev_ = -1;
    if (prev_ != dev) PAES_CK(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev_ >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev_) cudaSetDevice(prev_);
  }

 private:
  int prev_ = -1;
};

// ------------------------------------------------------------ host copy team
// Persistent threads for parallel host memcpy (the staged ring copies every
// piece in and out; a single core moves ~15 GB/s, and spawning a thread team
// per piece cost ~0.5 ms per 10 MiB piece).  copy() is blocking and splits
// the range over the team, the caller doing the first part; calls on one
// team serialise.  Workers are bound to the device's NUMA node.
class CopyTeam {
 public:
  CopyTeam(unsigned threads, int dev);
  ~CopyTeam();
  CopyTeam(const CopyTeam&) = delete;
  CopyTeam& operator=(const CopyTeam&) = delete;
  void copy(std::uint8_t* dst, const std::uint8_t* src, std::uint64_t n);

 private:
  void worker(unsigned idx, int dev);
  std::mutex call_mu_;  // one copy() at a time
  std::mutex mu_;
  std::condition_variable go_, done_;
  std::vector<std::thread> th_;
  std::uint8_t* dst_ = nullptr;
  const std::uint8_t* src_ = nullptr;
  std::uint64_t n_ = 0, step_ = 0;
  std::uint64_t gen_ = 0;
  unsigned pending_ = 0;
  bool stop_ = false;
};

// ------------------------------------------------------------ device context
struct DevCtx {
  int id = -1;
  std::atomic<bool> ready{false};  // set once, after every field below is initialised
  int sm_count = 0;
  std::mutex mu;  // serialises host-pointer pipelines / status words on this device
  std::vector<cudaStream_t> st;
  std::vector<std::uint8_t*> dbuf;  // chunk + 16 bytes each
  std::vector<std::uint8_t*> hbuf;  // pinned staging for the file path, hbuf_bytes + 16 each (ensure_host_ring)
  std::uint64_t hbuf_bytes = 0;
  // staged ring for pageable host buffers: pinned input and output slots
  // (kStagedSlot bytes + 16 each) and one copy team per direction
  std::vector<std::uint8_t*> sin_buf, sout_buf;
  std::unique_ptr<CopyTeam> team_in, team_out;
  std::vector<std::uint8_t*> obuf;  // second device ring (batch output spans), chunk + 16 each, lazy
  std::vector<std::uint8_t*> dsc;   // [0]: the host batch's device descriptor image (all groups), lazy, grow-only
  std::vector<std::size_t> dsc_cap;
  std::vector<cudaEvent_t> ev;
  // per slot, for the pinned ring's three queues: copy-in done, kernel done,
  // copy-out done (slot free)
  std::vector<cudaEvent_t> ev_in, ev_k, ev_out;
  std::uint64_t chunk = 0;
  std::uint32_t* h_status = nullptr;  // pinned, mapped; word 0 for host-pointer calls (d.mu held)
  std::uint32_t* m_status = nullptr;  // device alias of h_status: a one-shot check writes it directly
  std::mutex slot_mu;                 // guards free_slots
  std::vector<int> free_slots;        // status words 1.. for concurrent device-pointer final decrypts
  unsigned long long* d_acc = nullptr;
  unsigned long long* h_acc = nullptr;  // pinned
};

constexpr int kMaxDev = 64;

int visible_devices();
// Lazily initialised context of device `id` (throws CudaFail ENODEV).
DevCtx& device(int id);

// A status word of its own for one device-pointer final decrypt, so
// concurrent decrypts on different streams do not serialise on d.mu for the
// length of their kernels.  Falls back to word 0 under d.mu if all are busy.
class StatusSlot {
 public:
  explicit StatusSlot(DevCtx& d);
  ~StatusSlot();
  std::uint32_t* host() const { return d_.h_status + idx_; }
  std::uint32_t* dev() const { return d_.m_status + idx_; }

 private:
  DevCtx& d_;
  int idx_ = 0;
  std::unique_lock<std::mutex> fallback_;
};
// Pipeline buffers (device ring, optional pinned host ring); d.mu held.
void ensure_pipeline(DevCtx& d, bool need_host);
// The file path's pinned host slots, sized to the job's piece instead of the
// device slot: grow-only, `bytes` rounded up to a power of two between 16 MiB
// and the configured chunk.  Call after ensure_pipeline(d, false); d.mu held.
void ensure_host_ring(DevCtx& d, std::uint64_t bytes);
// Pins the calling library-owned thread (and the threads it spawns) to the
// CPUs of the device's NUMA node; a no-op where sysfs reports no node.
void bind_thread_to_device_numa(int dev);
// Pinned host <-> device copies whose bulk runs on 4 KiB-aligned host
// addresses: a head copy up to the next page boundary, then the rest.  With
// H2D and D2H in flight together (the ring), copies that start mid-page cost
// ~9 % of the PCIe rate (scripts/host_align_probe.py: 43.0 vs 47.2 GB/s);
// alone they do not (scripts/copy_align_probe.cu).
cudaError_t copy_h2d_aligned(void* dev, const void* host, std::uint64_t n, cudaStream_t s);
cudaError_t copy_d2h_aligned(void* host, const void* dev, std::uint64_t n, cudaStream_t s);

// Drains a device's ring streams when its scope is left by an exception: the
// copies and kernels already queued still target the caller's buffers and the
// ring's slots, so returning an error code before they finish would hand the
// caller buffers under live DMA.
struct QuiesceOnThrow {
  DevCtx& d;
  int depth = std::uncaught_exceptions();
  ~QuiesceOnThrow() {
    if (std::uncaught_exceptions() > depth)
      for (auto s : d.st) cudaStreamSynchronize(s);
  }
};
// Persistent host threads for multi-shard calls (a fresh
// std::thread per shard per call cost tens of microseconds).  run() hands
// shard k to pool thread k, which binds itself to the NUMA node of the
// device it serves (re-binding only when that changes), and returns when
// every shard is done.  Multi-shard calls from several host threads take
// turns; they would serialise on the devices' locks anyway.  f must not
// throw (callers wrap their shard work in guarded()).
class ShardPool {
 public:
  void run(const std::vector<int>& devs, const std::function<void(std::size_t)>& f);

 private:
  struct Worker {
    std::thread th;
    std::mutex mu;
    std::condition_variable cv;
    std::function<void()> job;
    int dev = -1;
  };
  void loop(Worker* w);
  std::mutex call_mu_;
  std::vector<std::unique_ptr<Worker>> workers_;
  std::mutex done_mu_;
  std::condition_variable done_cv_;
  std::size_t pending_ = 0;
};
// The process-wide pool (never destroyed: its threads park until exit).
ShardPool& shard_pool();

// The devices host-pointer calls shard over (first `ngpus`; 0 = all listed,
// at most one per kMinShardBytes of `len`).
std::vector<int> device_list(int ngpus);
std::vector<int> shard_devices(int ngpus, std::uint64_t len);
void set_device_list(const std::vector<int>& ids);
void set_pipeline_config(std::uint64_t chunk_bytes, int streams);
void set_zero_copy_max(std::uint64_t bytes);

// ------------------------------------------------------------ pieces
// A transform over one contiguous range: whole input blocks, plus (encrypt,
// final) the always-pad block built from `tail` trailing bytes, plus
// (decrypt, final) a trailer check on the last block.
struct Range {
  bool dec = false;
  bool pad = false;        // encrypt: append the PKCS#7 block
  bool check_pad = false;  // decrypt: validate the trailer
  std::uint64_t in_len = 0;
};

// In and out may be the same buffer (aes.hpp:84-85: "may alias exactly") or
// disjoint; a partial overlap would let one CTA overwrite input another has
// not read yet, so it is rejected (std::invalid_argument) before any device
// work.  Host-only: safe to call without a GPU.
void check_alias(const void* in, std::uint64_t in_len, const void* out, std::uint64_t out_len);

EcbArgs make_args(const Range& r, const std::uint8_t* in, std::uint8_t* out, std::uint64_t in_len, bool last,
                  const KeyWords& kw, std::uint32_t* status);
std::uint64_t piece_size(std::uint64_t len, std::uint64_t chunk, int streams);
// Host buffers on the device list: plan_chunks shards, one thread per shard.
int host_transform(int dir, const std::uint8_t* in, std::uint64_t len, bool is_final, const std::uint8_t* rk,
                   std::uint8_t* out, std::uint64_t* out_len, int ngpus);

}  // namespace paes_b200::rt
