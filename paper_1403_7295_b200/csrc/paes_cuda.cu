// paes_cuda.cu -- the C ABI (include/paes_cuda.h) and the host runtime around
// the sm_100a kernels: per-device contexts, the multi-stream host<->device
// pipeline, the multi-GPU block-range sharder and the file pipeline.
//
// Reference boundary: aes::encrypt_ecb/decrypt_ecb
// (aes.hpp:86-89), paes::encrypt_chunk/decrypt_chunk (exec.hpp:61-65) and
// run_job's strategy dispatch (exec.cpp:340-347).  Exceptions become codes:
// std::invalid_argument -> PAES_EINVAL, PaddingError -> PAES_EBADMSG,
// IoError -> PAES_EIO, WorkerError -> PAES_EWORKER, CUDA -> PAES_ECUDA.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "../../include/paes_cuda.h"
#include "host_rules.hpp"
#include "launch.hpp"

using namespace paes_b200;

namespace {

thread_local std::string t_err;

int fail(int code, const std::string& msg) {
  t_err = msg;
  return code;
}

struct CudaFail {
  int code;
  std::string msg;
};

#define PAES_CK(call)                                                                           \
  do {                                                                                          \
    const cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess) throw CudaFail{PAES_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)}; \
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

// ------------------------------------------------------------ device context
struct DevCtx {
  int id = -1;
  bool ready = false;
  int sm_count = 0;
  std::mutex mu;  // serialises host-pointer pipelines / status words on this device
  std::vector<cudaStream_t> st;
  std::vector<std::uint8_t*> dbuf;  // chunk + 16 bytes each
  std::vector<std::uint8_t*> hbuf;  // pinned staging for the file path
  std::vector<cudaEvent_t> ev;
  std::uint64_t chunk = 0;
  std::uint32_t* d_status = nullptr;
  std::uint32_t* h_status = nullptr;  // pinned
  unsigned long long* d_acc = nullptr;
  unsigned long long* h_acc = nullptr;  // pinned
};

constexpr int kMaxDev = 64;
DevCtx g_dev[kMaxDev];
std::mutex g_cfg_mu;
std::vector<int> g_devices;  // empty = all visible
std::uint64_t g_chunk = 64ull << 20;  // scripts/pcie_probe.py: 64-128 MiB pieces reach ~94% of concurrent H2D+D2H
int g_streams = 3;

int visible_devices() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

// Lazily initialise a device: kernel attributes, status words.
DevCtx& device(int id) {
  const int n = visible_devices();
  if (id < 0 || id >= n || id >= kMaxDev)
    throw CudaFail{PAES_ENODEV, "no such CUDA device: " + std::to_string(id) + " (visible: " + std::to_string(n) + ")"};
  DevCtx& d = g_dev[id];
  std::lock_guard<std::mutex> lk(d.mu);
  if (!d.ready) {
    DeviceGuard g(id);
    PAES_CK(cudaDeviceGetAttribute(&d.sm_count, cudaDevAttrMultiProcessorCount, id));
    PAES_CK(prepare_kernels());
    PAES_CK(cudaMalloc(&d.d_status, 4096));
    PAES_CK(cudaMallocHost(&d.h_status, 4096));
    PAES_CK(cudaMalloc(&d.d_acc, 64));
    PAES_CK(cudaMallocHost(&d.h_acc, 64));
    d.id = id;
    d.ready = true;
  }
  return d;
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
  if (d.chunk != chunk || static_cast<int>(d.st.size()) != ns) {
    for (auto p : d.dbuf) cudaFree(p);
    for (auto p : d.hbuf) cudaFreeHost(p);
    for (auto s : d.st) cudaStreamDestroy(s);
    for (auto e : d.ev) cudaEventDestroy(e);
    d.dbuf.clear();
    d.hbuf.clear();
    d.st.clear();
    d.ev.clear();
    d.chunk = chunk;
    for (int i = 0; i < ns; ++i) {
      cudaStream_t s;
      PAES_CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
      d.st.push_back(s);
      cudaEvent_t e;
      PAES_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      d.ev.push_back(e);
      std::uint8_t* p = nullptr;
      PAES_CK(cudaMalloc(&p, chunk + 16));
      d.dbuf.push_back(p);
    }
  }
  if (need_host && d.hbuf.empty()) {
    for (int i = 0; i < ns; ++i) {
      std::uint8_t* p = nullptr;
      PAES_CK(cudaMallocHost(&p, d.chunk + 16));
      d.hbuf.push_back(p);
    }
  }
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

// Piece size for a range: the staging chunk, but small enough that even a
// short range is split into ~2 pieces per stream so copy-in, kernel and
// copy-out still overlap (a single 64 MiB piece would serialise them).
std::uint64_t piece_size(std::uint64_t len, std::uint64_t chunk, int streams) {
  const std::uint64_t floor_piece = std::min<std::uint64_t>(4ull << 20, chunk);
  const std::uint64_t p = (len / (2ull * static_cast<std::uint64_t>(streams)) + 15) & ~std::uint64_t(15);
  return std::clamp(p, floor_piece, chunk);
}

// Host range on one device through the stream ring (d.mu held).  Returns the
// number of output bytes (decrypt+check: unpadded).
// Small host ranges (<= kSmallBytes): one memcpy into a mapped pinned buffer,
// ONE kernel that reads and writes that host buffer over PCIe (zero-copy),
// one sync, one memcpy out.  Replaces H2D + launch + D2H (three commands and
// their latencies) for the short messages of config 3 / encrypt_bytes.
constexpr std::uint64_t kSmallBytes = 1ull << 20;

struct SmallBuf {
  std::uint8_t* host = nullptr;  // mapped pinned, kSmallBytes + 32
  std::uint8_t* dev = nullptr;   // its device alias
  std::uint32_t* status_host = nullptr;
  std::uint32_t* status_dev = nullptr;
};
SmallBuf g_small[kMaxDev];

std::uint64_t run_small(DevCtx& d, const Range& r, const std::uint8_t* in, std::uint8_t* out, const KeyWords& kw) {
  SmallBuf& sb = g_small[d.id];
  if (!sb.host) {
    void* p = nullptr;
    PAES_CK(cudaHostAlloc(&p, kSmallBytes + 4096, cudaHostAllocMapped | cudaHostAllocPortable));
    sb.host = static_cast<std::uint8_t*>(p);
    PAES_CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&sb.dev), p, 0));
    sb.status_host = reinterpret_cast<std::uint32_t*>(sb.host + kSmallBytes + 2048);
    sb.status_dev = reinterpret_cast<std::uint32_t*>(sb.dev + kSmallBytes + 2048);
  }
  if (r.in_len) std::memcpy(sb.host, in, r.in_len);
  *sb.status_host = 0xffffffffu;  // sentinel: unchecked => PaddingError
  EcbArgs a = make_args(r, sb.dev, sb.dev, r.in_len, true, kw, sb.status_dev);
  PAES_CK(launch_ecb(r.dec, a, d.sm_count, d.st[0]));
  PAES_CK(cudaStreamSynchronize(d.st[0]));
  std::uint64_t olen = a.nblocks * 16;
  if (olen) std::memcpy(out, sb.host, olen);
  if (r.check_pad) {
    const std::uint32_t k = *reinterpret_cast<volatile std::uint32_t*>(sb.status_host);
    if (k == 0xffffffffu) throw PaddingError("unpad: invalid pad bytes");
    olen -= k;
  }
  return olen;
}

bool is_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// memcpy split over host threads (a single core moves ~10 GB/s; the pinned
// slots are fed at PCIe rate).
void par_copy(std::uint8_t* dst, const std::uint8_t* src, std::uint64_t n) {
  constexpr std::uint64_t kGrain = 8ull << 20;
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const std::uint64_t parts = std::min<std::uint64_t>(std::min(hw, 8u), (n + kGrain - 1) / kGrain);
  if (parts <= 1) {
    if (n) std::memcpy(dst, src, n);
    return;
  }
  const std::uint64_t step = ((n / parts) + 4095) & ~std::uint64_t(4095);
  std::vector<std::thread> pool;
  for (std::uint64_t i = 1; i < parts; ++i) {
    const std::uint64_t b = std::min(n, i * step), e = std::min(n, (i + 1) * step);
    if (b < e) pool.emplace_back([=] { std::memcpy(dst + b, src + b, e - b); });
  }
  std::memcpy(dst, src, std::min(n, step));
  for (auto& t : pool) t.join();
}

// Pageable host buffers (std::vector, Python bytes): stage through the pinned
// slot ring ourselves -- copy piece k in while the GPU works on earlier
// pieces, copy each finished piece out when its slot comes round again.  The
// driver's own staging of pageable cudaMemcpyAsync serialises at ~7 GB/s.
std::uint64_t run_host_range_staged(DevCtx& d, const Range& r, const std::uint8_t* in, std::uint8_t* out,
                                    const KeyWords& kw) {
  ensure_pipeline(d, true);
  const int S = static_cast<int>(d.st.size());
  const std::uint64_t C = piece_size(r.in_len, d.chunk, S);
  const std::uint64_t npieces = std::max<std::uint64_t>(1, (r.in_len + C - 1) / C);
  std::vector<std::int64_t> pend_off(S, -1);
  std::vector<std::uint64_t> pend_len(S, 0);
  auto drain = [&](int s) {
    if (pend_off[s] < 0) return;
    PAES_CK(cudaEventSynchronize(d.ev[s]));
    par_copy(out + pend_off[s], d.hbuf[s], pend_len[s]);
    pend_off[s] = -1;
  };
  std::uint64_t out_total = 0;
  for (std::uint64_t k = 0; k < npieces; ++k) {
    const int s = static_cast<int>(k % S);
    drain(s);
    const std::uint64_t off = k * C;
    const std::uint64_t len = std::min<std::uint64_t>(C, r.in_len - off);
    const bool last = k + 1 == npieces;
    par_copy(d.hbuf[s], in + off, len);
    EcbArgs a = make_args(r, d.dbuf[s], d.dbuf[s], len, last, kw, d.d_status);
    if (len) PAES_CK(cudaMemcpyAsync(d.dbuf[s], d.hbuf[s], len, cudaMemcpyHostToDevice, d.st[s]));
    if (a.check_pad) PAES_CK(cudaMemsetAsync(d.d_status, 0xff, 4, d.st[s]));
    PAES_CK(launch_ecb(r.dec, a, d.sm_count, d.st[s]));
    const std::uint64_t olen = a.nblocks * 16;
    if (olen) PAES_CK(cudaMemcpyAsync(d.hbuf[s], d.dbuf[s], olen, cudaMemcpyDeviceToHost, d.st[s]));
    if (last && a.check_pad) PAES_CK(cudaMemcpyAsync(d.h_status, d.d_status, 4, cudaMemcpyDeviceToHost, d.st[s]));
    PAES_CK(cudaEventRecord(d.ev[s], d.st[s]));
    pend_off[s] = static_cast<std::int64_t>(off);
    pend_len[s] = olen;
    out_total = off + olen;
  }
  for (int s = 0; s < S; ++s) drain(s);
  if (r.check_pad) {
    const std::uint32_t k = *d.h_status;
    if (k == 0xffffffffu) throw PaddingError("unpad: invalid pad bytes");
    out_total -= k;
  }
  return out_total;
}

std::uint64_t run_host_range(DevCtx& d, const Range& r, const std::uint8_t* in, std::uint8_t* out, const KeyWords& kw) {
  DeviceGuard g(d.id);
  ensure_pipeline(d, false);
  if (r.in_len <= std::min(kSmallBytes, d.chunk)) return run_small(d, r, in, out, kw);
  if (!is_pinned(in) || !is_pinned(out)) return run_host_range_staged(d, r, in, out, kw);
  const int S = static_cast<int>(d.st.size());
  const std::uint64_t C = piece_size(r.in_len, d.chunk, S);
  const std::uint64_t npieces = std::max<std::uint64_t>(1, (r.in_len + C - 1) / C);
  std::uint64_t out_total = 0;
  for (std::uint64_t k = 0; k < npieces; ++k) {
    const int s = static_cast<int>(k % S);
    const std::uint64_t off = k * C;
    const std::uint64_t len = std::min<std::uint64_t>(C, r.in_len - off);
    const bool last = k + 1 == npieces;
    EcbArgs a = make_args(r, d.dbuf[s], d.dbuf[s], len, last, kw, d.d_status);
    if (len) PAES_CK(cudaMemcpyAsync(d.dbuf[s], in + off, len, cudaMemcpyHostToDevice, d.st[s]));
    if (a.check_pad) PAES_CK(cudaMemsetAsync(d.d_status, 0xff, 4, d.st[s]));  // sentinel: unchecked => PaddingError
    PAES_CK(launch_ecb(r.dec, a, d.sm_count, d.st[s]));
    const std::uint64_t olen = a.nblocks * 16;
    if (olen) PAES_CK(cudaMemcpyAsync(out + off, d.dbuf[s], olen, cudaMemcpyDeviceToHost, d.st[s]));
    if (last && a.check_pad)
      PAES_CK(cudaMemcpyAsync(d.h_status, d.d_status, 4, cudaMemcpyDeviceToHost, d.st[s]));
    out_total = off + olen;
  }
  for (auto s : d.st) PAES_CK(cudaStreamSynchronize(s));
  if (r.check_pad) {
    const std::uint32_t k = *d.h_status;
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
  const auto devs = device_list(ngpus);
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
      std::lock_guard<std::mutex> lk(d.mu);
      produced[i] = run_host_range(d, r, in + c.offset, out + c.offset, kw);
      return PAES_OK;
    });
    if (codes[i]) msgs[i] = t_err;
  };
  if (plan.size() == 1) {
    work(0);
  } else {
    std::vector<std::thread> pool;
    for (std::size_t i = 0; i < plan.size(); ++i) pool.emplace_back(work, i);
    for (auto& t : pool) t.join();
  }
  for (std::size_t i = 0; i < plan.size(); ++i)
    if (codes[i]) return fail(codes[i], msgs[i]);
  std::uint64_t total = 0;
  for (auto p : produced) total += p;
  if (out_len) *out_len = total;
  return PAES_OK;
}

}  // namespace

// ============================================================ C ABI
extern "C" {

const char* paes_cuda_last_error(void) { return t_err.c_str(); }

const char* paes_cuda_version(void) { return "paes_cuda 0.1 sm_100a (T-table smem x32, PRMT-addressed)"; }

int paes_cuda_device_count(void) { return visible_devices(); }

int paes_cuda_set_devices(const int* ids, int n) {
  return guarded([&] {
    if (n < 0 || (n > 0 && !ids)) throw std::invalid_argument("bad device list");
    const int vis = visible_devices();
    for (int i = 0; i < n; ++i)
      if (ids[i] < 0 || ids[i] >= vis) throw CudaFail{PAES_ENODEV, "no such CUDA device: " + std::to_string(ids[i])};
    std::lock_guard<std::mutex> lk(g_cfg_mu);
    g_devices.assign(ids, ids + n);
    return PAES_OK;
  });
}

int paes_cuda_set_pipeline(uint64_t chunk_bytes, int streams) {
  return guarded([&] {
    if (chunk_bytes % 16 != 0) throw std::invalid_argument("chunk_bytes must be a multiple of 16");
    if (streams < 0) throw std::invalid_argument("streams must be >= 0");
    std::lock_guard<std::mutex> lk(g_cfg_mu);
    if (chunk_bytes) g_chunk = chunk_bytes;
    if (streams) g_streams = streams;
    return PAES_OK;
  });
}

int paes_cuda_expand_key(const uint8_t key[16], uint8_t rk[176]) {
  return guarded([&] {
    if (!key || !rk) throw std::invalid_argument("null key");
    expand_key(key, rk);
    return PAES_OK;
  });
}

static int64_t plan_out(const std::vector<Chunk>& p, paes_chunk_spec* out, uint64_t cap) {
  for (std::size_t i = 0; i < p.size() && i < cap; ++i)
    out[i] = paes_chunk_spec{p[i].offset, p[i].raw_len, p[i].padded_len, p[i].is_final ? 1 : 0, 0};
  return static_cast<int64_t>(p.size());
}

int64_t paes_cuda_plan_chunks(uint64_t total_len, uint32_t workers, paes_chunk_spec* out, uint64_t cap) {
  int64_t n = 0;
  const int rc = guarded([&] {
    n = plan_out(plan_chunks(total_len, workers), out, out ? cap : 0);
    return PAES_OK;
  });
  return rc ? rc : n;
}

int64_t paes_cuda_plan_decrypt_chunks(uint64_t cipher_len, uint32_t workers, paes_chunk_spec* out, uint64_t cap) {
  int64_t n = 0;
  const int rc = guarded([&] {
    n = plan_out(plan_decrypt_chunks(cipher_len, workers), out, out ? cap : 0);
    return PAES_OK;
  });
  return rc ? rc : n;
}

int64_t paes_cuda_pad_final(const uint8_t* raw, uint64_t len, uint8_t* out) {
  if ((len && !raw) || !out) return fail(PAES_EINVAL, "null buffer");
  const uint64_t k = 16 - len % 16;
  if (len && raw != out) std::memmove(out, raw, len);
  std::memset(out + len, static_cast<int>(k), k);
  return static_cast<int64_t>(len + k);
}

int64_t paes_cuda_unpad_final(const uint8_t* padded, uint64_t len) {
  int64_t n = 0;
  const int rc = guarded([&] {
    if (len && !padded) throw std::invalid_argument("null buffer");
    n = static_cast<int64_t>(unpad_final(padded, len));
    return PAES_OK;
  });
  return rc ? rc : n;
}

int paes_cuda_ecb(int dir, const uint8_t* in, uint8_t* out, uint64_t len, const uint8_t rk[176], int ngpus) {
  return guarded([&] {
    if (len % 16 != 0) throw std::invalid_argument("ecb: length must be a multiple of 16 and match output");
    return host_transform(dir, in, len, false, rk, out, nullptr, ngpus);
  });
}

int paes_cuda_chunk(int dir, const uint8_t* in, uint64_t len, int is_final, const uint8_t rk[176], uint8_t* out,
                    uint64_t* out_len, int ngpus) {
  return guarded([&] { return host_transform(dir, in, len, is_final != 0, rk, out, out_len, ngpus); });
}

int paes_cuda_ecb_device(int dir, const void* d_in, void* d_out, uint64_t len, const uint8_t rk[176], int device_id,
                         void* stream) {
  return guarded([&] {
    if (dir != PAES_ENCRYPT && dir != PAES_DECRYPT) throw std::invalid_argument("bad dir");
    if (len % 16 != 0) throw std::invalid_argument("ecb: length must be a multiple of 16 and match output");
    if (!rk) throw std::invalid_argument("null round keys");
    if (len == 0) return PAES_OK;
    if (!d_in || !d_out) throw std::invalid_argument("null device buffer");
    DevCtx& d = device(device_id);
    DeviceGuard g(device_id);
    const bool dec = dir == PAES_DECRYPT;
    Range r;
    r.dec = dec;
    EcbArgs a = make_args(r, static_cast<const std::uint8_t*>(d_in), static_cast<std::uint8_t*>(d_out), len, true,
                          dec ? dec_key_words(rk) : enc_key_words(rk), nullptr);
    PAES_CK(launch_ecb(dec, a, d.sm_count, static_cast<cudaStream_t>(stream)));
    return PAES_OK;
  });
}

int paes_cuda_chunk_device(int dir, const void* d_in, uint64_t len, int is_final, const uint8_t rk[176], void* d_out,
                           uint64_t* out_len, int device_id, void* stream) {
  return guarded([&] {
    if (dir != PAES_ENCRYPT && dir != PAES_DECRYPT) throw std::invalid_argument("bad dir");
    if (!rk) throw std::invalid_argument("null round keys");
    const bool dec = dir == PAES_DECRYPT;
    const bool final = is_final != 0;
    if (!final && len % 16 != 0) throw std::invalid_argument("non-final chunk length must be a multiple of 16");
    if (dec && len % 16 != 0) throw std::invalid_argument("decrypt: length must be a multiple of 16");
    if (dec && final && len == 0) throw PaddingError("unpad: length must be a non-zero multiple of 16");
    Range r;
    r.dec = dec;
    r.pad = !dec && final;
    r.check_pad = dec && final;
    if (len == 0 && !r.pad) {
      if (out_len) *out_len = 0;
      return PAES_OK;
    }
    if ((len && !d_in) || !d_out) throw std::invalid_argument("null device buffer");
    DevCtx& d = device(device_id);
    DeviceGuard g(device_id);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (!r.check_pad) {
      EcbArgs a = make_args(r, static_cast<const std::uint8_t*>(d_in), static_cast<std::uint8_t*>(d_out), len, true,
                            dec ? dec_key_words(rk) : enc_key_words(rk), nullptr);
      PAES_CK(launch_ecb(dec, a, d.sm_count, s));
      if (out_len) *out_len = a.nblocks * 16;
      return PAES_OK;
    }
    std::lock_guard<std::mutex> lk(d.mu);
    EcbArgs a = make_args(r, static_cast<const std::uint8_t*>(d_in), static_cast<std::uint8_t*>(d_out), len, true,
                          dec_key_words(rk), d.d_status);
    PAES_CK(cudaMemsetAsync(d.d_status, 0xff, 4, s));
    PAES_CK(launch_ecb(true, a, d.sm_count, s));
    PAES_CK(cudaMemcpyAsync(d.h_status, d.d_status, 4, cudaMemcpyDeviceToHost, s));
    PAES_CK(cudaStreamSynchronize(s));
    const std::uint32_t k = *d.h_status;
    if (k == 0xffffffffu) throw PaddingError("unpad: invalid pad bytes");
    if (out_len) *out_len = len - k;
    return PAES_OK;
  });
}

}  // extern "C"

// ------------------------------------------------------------ batch (config 5)
namespace {

// Host image of a batch: BatchMsg[n] | KeyWords[n] (| status words when the
// trailers are checked).  Validation mirrors encrypt_chunk / decrypt_chunk per
// message (exec.cpp:375-392).
struct BatchImage {
  bool dec = false, check = false;
  std::uint32_t n = 0;
  unsigned long long total_tiles = 0;  // warp tiles (each message owns whole tiles)
  std::size_t msg_bytes = 0, keys_off = 0, image_bytes = 0, status_off = 0, total_bytes = 0;
  std::vector<std::uint64_t> lens;
  std::vector<std::uint32_t> nblocks;
};

BatchImage plan_batch(int dir, const uint64_t* in_off, const uint64_t* out_off, const uint64_t* lens,
                      const uint8_t* rks, uint32_t n, int pad) {
  if (dir != PAES_ENCRYPT && dir != PAES_DECRYPT) throw std::invalid_argument("bad dir");
  if (n && (!in_off || !out_off || !lens || !rks)) throw std::invalid_argument("null batch descriptor");
  BatchImage b;
  b.dec = dir == PAES_DECRYPT;
  b.check = b.dec && pad;
  b.n = n;
  b.msg_bytes = sizeof(BatchMsg) * n;
  b.keys_off = (b.msg_bytes + 255) & ~std::size_t(255);  // 16-byte key loads need alignment
  b.image_bytes = b.keys_off + sizeof(KeyWords) * n;
  b.status_off = (b.image_bytes + 255) & ~std::size_t(255);
  b.total_bytes = b.status_off + (b.check ? 4ull * n : 0);
  b.lens.assign(lens, lens + n);
  b.nblocks.resize(n);
  for (uint32_t i = 0; i < n; ++i) {
    if (in_off[i] % 16 || out_off[i] % 16) throw std::invalid_argument("batch offsets must be multiples of 16");
    if ((b.dec || !pad) && lens[i] % 16) throw std::invalid_argument("message length must be a multiple of 16");
    if (b.check && lens[i] == 0) throw PaddingError("unpad: length must be a non-zero multiple of 16");
    const unsigned long long nb = lens[i] / 16 + ((pad && !b.dec) ? 1 : 0);
    if (nb > 0xffffffffull) throw std::invalid_argument("message too large for the batch path");
    b.nblocks[i] = static_cast<std::uint32_t>(nb);
    b.total_tiles += (nb + batch_tile_blocks() - 1) / batch_tile_blocks();
  }
  return b;
}

void write_batch_image(const BatchImage& b, const uint64_t* in_off, const uint64_t* out_off, const uint8_t* rks,
                       std::uint8_t* dst) {
  auto* msgs = reinterpret_cast<BatchMsg*>(dst);
  auto* keys = reinterpret_cast<KeyWords*>(dst + b.keys_off);
  unsigned long long tile = 0;
  for (uint32_t i = 0; i < b.n; ++i) {
    BatchMsg m{};
    m.in_off = in_off[i];
    m.out_off = out_off[i];
    m.first_tile = tile;
    m.nfull = b.lens[i] / 16;
    m.tail_len = static_cast<std::uint32_t>(b.lens[i] % 16);
    m.nblocks = b.nblocks[i];
    tile += (m.nblocks + batch_tile_blocks() - 1) / batch_tile_blocks();
    msgs[i] = m;
    keys[i] = b.dec ? dec_key_words(rks + 176ull * i) : enc_key_words(rks + 176ull * i);
  }
}

BatchArgs batch_args(const BatchImage& b, const void* d_in, void* d_out, std::uint8_t* dd) {
  BatchArgs a{};
  a.in = static_cast<const std::uint8_t*>(d_in);
  a.out = static_cast<std::uint8_t*>(d_out);
  a.msgs = reinterpret_cast<const BatchMsg*>(dd);
  a.keys = reinterpret_cast<const std::uint32_t*>(dd + b.keys_off);
  a.status = b.check ? reinterpret_cast<std::uint32_t*>(dd + b.status_off) : nullptr;
  a.total_tiles = b.total_tiles;
  a.nmsg = b.n;
  a.check_pad = b.check ? 1u : 0u;
  return a;
}

void finish_lengths(const BatchImage& b, const std::uint32_t* status, uint64_t* out_lens) {
  if (!b.check) {
    if (out_lens)
      for (uint32_t i = 0; i < b.n; ++i) out_lens[i] = static_cast<uint64_t>(b.nblocks[i]) * 16;
    return;
  }
  bool bad = false;
  for (uint32_t i = 0; i < b.n; ++i) {
    const bool ok = status[i] != 0xffffffffu;
    bad |= !ok;
    if (out_lens) out_lens[i] = ok ? b.lens[i] - status[i] : UINT64_MAX;
  }
  if (bad) throw PaddingError("unpad: invalid pad bytes in one or more messages");
}

// Per-thread pinned staging for one-shot batches: the descriptor upload is a
// true async copy, and the buffer is reused once its previous copy is done.
struct Staging {
  std::uint8_t* p = nullptr;
  std::size_t cap = 0;
  int device = -1;
  cudaEvent_t ev = nullptr;
  ~Staging() {
    if (p) cudaFreeHost(p);
  }
};
thread_local Staging t_stage;

std::uint8_t* staging(std::size_t bytes, int device) {
  Staging& st = t_stage;
  if (st.ev && st.device == device) PAES_CK(cudaEventSynchronize(st.ev));
  if (st.device != device) {
    if (st.ev) cudaEventDestroy(st.ev);
    st.ev = nullptr;
    st.device = device;
  }
  if (!st.ev) PAES_CK(cudaEventCreateWithFlags(&st.ev, cudaEventDisableTiming));
  if (st.cap < bytes) {
    if (st.p) PAES_CK(cudaFreeHost(st.p));
    st.p = nullptr;
    st.cap = 0;
    PAES_CK(cudaMallocHost(&st.p, bytes));
    st.cap = bytes;
  }
  return st.p;
}

}  // namespace

struct paes_batch_plan {
  int device = -1;
  BatchImage img;
  std::uint8_t* dd = nullptr;        // device image
  std::uint32_t* h_status = nullptr;  // pinned
};

extern "C" {

int paes_cuda_ecb_batch(int dir, const void* d_in, void* d_out, const uint64_t* in_off, const uint64_t* out_off,
                        const uint64_t* lens, const uint8_t* rks, uint32_t n, int pad, uint64_t* out_lens,
                        int device_id, void* stream) {
  return guarded([&] {
    const BatchImage b = plan_batch(dir, in_off, out_off, lens, rks, n, pad);
    if (n == 0) return PAES_OK;
    if (!d_in || !d_out) throw std::invalid_argument("null device buffer");
    DevCtx& d = device(device_id);
    DeviceGuard dg(device_id);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    std::uint8_t* host = staging(b.total_bytes, device_id);
    write_batch_image(b, in_off, out_off, rks, host);
    std::uint8_t* dd = nullptr;
    PAES_CK(cudaMallocAsync(reinterpret_cast<void**>(&dd), b.total_bytes, s));
    PAES_CK(cudaMemcpyAsync(dd, host, b.image_bytes, cudaMemcpyHostToDevice, s));
    PAES_CK(cudaEventRecord(t_stage.ev, s));
    PAES_CK(launch_batch(b.dec, batch_args(b, d_in, d_out, dd), d.sm_count, s));
    if (b.check) {
      auto* st = reinterpret_cast<std::uint32_t*>(host + b.status_off);
      PAES_CK(cudaMemcpyAsync(st, dd + b.status_off, 4ull * n, cudaMemcpyDeviceToHost, s));
      PAES_CK(cudaFreeAsync(dd, s));
      PAES_CK(cudaStreamSynchronize(s));
      finish_lengths(b, st, out_lens);
    } else {
      PAES_CK(cudaFreeAsync(dd, s));
      finish_lengths(b, nullptr, out_lens);
    }
    return PAES_OK;
  });
}

int paes_cuda_batch_plan_create(int dir, const uint64_t* in_off, const uint64_t* out_off, const uint64_t* lens,
                                const uint8_t* rks, uint32_t n, int pad, int device_id, paes_batch_plan** plan) {
  return guarded([&] {
    if (!plan) throw std::invalid_argument("null plan pointer");
    *plan = nullptr;
    auto p = std::make_unique<paes_batch_plan>();
    p->img = plan_batch(dir, in_off, out_off, lens, rks, n, pad);
    p->device = device_id;
    device(device_id);
    DeviceGuard dg(device_id);
    if (n) {
      std::vector<std::uint8_t> host(p->img.image_bytes);
      write_batch_image(p->img, in_off, out_off, rks, host.data());
      PAES_CK(cudaMalloc(reinterpret_cast<void**>(&p->dd), p->img.total_bytes));
      PAES_CK(cudaMemcpy(p->dd, host.data(), host.size(), cudaMemcpyHostToDevice));
      if (p->img.check) PAES_CK(cudaMallocHost(reinterpret_cast<void**>(&p->h_status), 4ull * n));
    }
    *plan = p.release();
    return PAES_OK;
  });
}

int paes_cuda_batch_plan_run(paes_batch_plan* plan, const void* d_in, void* d_out, uint64_t* out_lens, void* stream) {
  return guarded([&] {
    if (!plan) throw std::invalid_argument("null plan");
    const BatchImage& b = plan->img;
    if (b.n == 0) return PAES_OK;
    if (!d_in || !d_out) throw std::invalid_argument("null device buffer");
    DevCtx& d = device(plan->device);
    DeviceGuard dg(plan->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    PAES_CK(launch_batch(b.dec, batch_args(b, d_in, d_out, plan->dd), d.sm_count, s));
    if (b.check) {
      PAES_CK(cudaMemcpyAsync(plan->h_status, plan->dd + b.status_off, 4ull * b.n, cudaMemcpyDeviceToHost, s));
      PAES_CK(cudaStreamSynchronize(s));
      finish_lengths(b, plan->h_status, out_lens);
    } else {
      finish_lengths(b, nullptr, out_lens);
    }
    return PAES_OK;
  });
}

void paes_cuda_batch_plan_destroy(paes_batch_plan* plan) {
  if (!plan) return;
  if (plan->dd) {
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(plan->device);
    cudaFree(plan->dd);
    if (prev >= 0) cudaSetDevice(prev);
  }
  if (plan->h_status) cudaFreeHost(plan->h_status);
  delete plan;
}

// Host-pointer batch: consecutive messages are grouped into ~chunk-sized
// groups; per group one H2D of its input span, one batch launch over
// group-relative descriptors, one D2H of its output span, the groups
// round-robin over the device's stream ring so copies overlap compute.
int paes_cuda_batch_host(int dir, const uint8_t* h_in, uint8_t* h_out, const uint64_t* in_off, const uint64_t* out_off,
                         const uint64_t* lens, const uint8_t* rks, uint32_t n, int pad, uint64_t* out_lens,
                         int device_id) {
  return guarded([&] {
    const BatchImage all = plan_batch(dir, in_off, out_off, lens, rks, n, pad);
    if (n == 0) return PAES_OK;
    if (!h_in || !h_out) throw std::invalid_argument("null host buffer");
    DevCtx& d = device(device_id);
    DeviceGuard dg(device_id);
    std::lock_guard<std::mutex> lk(d.mu);
    ensure_pipeline(d, false);
    const std::uint64_t C = d.chunk;
    const int S = static_cast<int>(d.st.size());
    // groups of consecutive messages whose input and output spans stay <= C
    struct Group {
      std::uint32_t first, count;
      std::uint64_t in_lo, in_hi, out_lo, out_hi;
    };
    std::vector<Group> groups;
    for (std::uint32_t i = 0; i < n; ++i) {
      const std::uint64_t ilo = in_off[i], ihi = in_off[i] + lens[i];
      const std::uint64_t olo = out_off[i], ohi = out_off[i] + 16ull * all.nblocks[i];
      if (!groups.empty()) {
        Group& g = groups.back();
        const std::uint64_t nil = std::min(g.in_lo, ilo), nih = std::max(g.in_hi, ihi);
        const std::uint64_t nol = std::min(g.out_lo, olo), noh = std::max(g.out_hi, ohi);
        if (nih - nil <= C && noh - nol <= C) {
          g.count += 1;
          g.in_lo = nil, g.in_hi = nih, g.out_lo = nol, g.out_hi = noh;
          continue;
        }
      }
      groups.push_back({i, 1, ilo, ihi, olo, ohi});
    }
    // one pinned image for every group's descriptors (+ status words)
    std::vector<std::size_t> img_off(groups.size());
    std::vector<BatchImage> imgs;
    imgs.reserve(groups.size());
    std::size_t total = 0;
    std::vector<std::uint64_t> rin(n), rout(n);
    for (std::size_t k = 0; k < groups.size(); ++k) {
      const Group& g = groups[k];
      for (std::uint32_t i = g.first; i < g.first + g.count; ++i) {
        rin[i] = in_off[i] - g.in_lo;
        rout[i] = out_off[i] - g.out_lo;
      }
      imgs.push_back(plan_batch(dir, rin.data() + g.first, rout.data() + g.first, lens + g.first,
                                rks + 176ull * g.first, g.count, pad));
      img_off[k] = total;
      total += (imgs.back().total_bytes + 255) & ~std::size_t(255);
    }
    std::uint8_t* host = staging(total, device_id);
    for (std::size_t k = 0; k < groups.size(); ++k) {
      const Group& g = groups[k];
      write_batch_image(imgs[k], rin.data() + g.first, rout.data() + g.first, rks + 176ull * g.first,
                        host + img_off[k]);
    }
    for (std::size_t k = 0; k < groups.size(); ++k) {
      const Group& g = groups[k];
      const BatchImage& b = imgs[k];
      cudaStream_t s = d.st[k % S];
      std::uint8_t *din = nullptr, *dout = nullptr, *dd = nullptr;
      PAES_CK(cudaMallocAsync(reinterpret_cast<void**>(&din), std::max<std::uint64_t>(16, g.in_hi - g.in_lo), s));
      PAES_CK(cudaMallocAsync(reinterpret_cast<void**>(&dout), std::max<std::uint64_t>(16, g.out_hi - g.out_lo), s));
      PAES_CK(cudaMallocAsync(reinterpret_cast<void**>(&dd), b.total_bytes, s));
      if (g.in_hi > g.in_lo)
        PAES_CK(cudaMemcpyAsync(din, h_in + g.in_lo, g.in_hi - g.in_lo, cudaMemcpyHostToDevice, s));
      PAES_CK(cudaMemcpyAsync(dd, host + img_off[k], b.image_bytes, cudaMemcpyHostToDevice, s));
      PAES_CK(launch_batch(b.dec, batch_args(b, din, dout, dd), d.sm_count, s));
      PAES_CK(cudaMemcpyAsync(h_out + g.out_lo, dout, g.out_hi - g.out_lo, cudaMemcpyDeviceToHost, s));
      if (b.check)
        PAES_CK(cudaMemcpyAsync(host + img_off[k] + b.status_off, dd + b.status_off, 4ull * b.n,
                                cudaMemcpyDeviceToHost, s));
      PAES_CK(cudaFreeAsync(din, s));
      PAES_CK(cudaFreeAsync(dout, s));
      PAES_CK(cudaFreeAsync(dd, s));
    }
    for (auto s : d.st) PAES_CK(cudaStreamSynchronize(s));
    PAES_CK(cudaEventRecord(t_stage.ev, d.st[0]));
    bool bad = false;
    for (std::size_t k = 0; k < groups.size(); ++k) {
      const BatchImage& b = imgs[k];
      try {
        finish_lengths(b, b.check ? reinterpret_cast<const std::uint32_t*>(host + img_off[k] + b.status_off) : nullptr,
                       out_lens ? out_lens + groups[k].first : nullptr);
      } catch (const PaddingError&) {
        bad = true;
      }
    }
    if (bad) throw PaddingError("unpad: invalid pad bytes in one or more messages");
    return PAES_OK;
  });
}

int paes_cuda_sweep(uint64_t seed, uint64_t size, uint8_t* out) {
  return guarded([&] {
    if (size && !out) throw std::invalid_argument("null buffer");
    sweep(seed, size, out);
    return PAES_OK;
  });
}

int paes_cuda_batch_lengths(uint64_t seed, uint32_t n, uint64_t* lens) {
  return guarded([&] {
    if (n && !lens) throw std::invalid_argument("null buffer");
    batch_lengths(seed, n, lens);
    return PAES_OK;
  });
}

int paes_cuda_counter_fill(uint64_t seed, uint64_t offset, uint64_t size, uint8_t* out) {
  return guarded([&] {
    if (offset % 8) throw std::invalid_argument("offset must be a multiple of 8");
    if (size && !out) throw std::invalid_argument("null buffer");
    uint64_t wi = offset / 8;
    for (uint64_t off = 0; off < size; off += 8) {
      const uint64_t w = counter_word(seed, wi++);
      const uint64_t n = std::min<uint64_t>(8, size - off);
      std::memcpy(out + off, &w, n);  // little-endian host
    }
    return PAES_OK;
  });
}

int paes_cuda_counter_fill_device(uint64_t seed, uint64_t offset, uint64_t size, void* d_out, int device_id,
                                  void* stream) {
  return guarded([&] {
    if (offset % 8 || size % 8) throw std::invalid_argument("offset and size must be multiples of 8");
    if (size == 0) return PAES_OK;
    if (!d_out || reinterpret_cast<std::uintptr_t>(d_out) % 16) throw std::invalid_argument("d_out must be 16-byte aligned");
    DevCtx& d = device(device_id);
    DeviceGuard g(device_id);
    PAES_CK(launch_counter_fill(seed, offset / 8, size / 8, d_out, d.sm_count, static_cast<cudaStream_t>(stream)));
    return PAES_OK;
  });
}

int paes_cuda_checksum(const uint8_t* buf, uint64_t len, uint64_t base_word, uint64_t* out) {
  return guarded([&] {
    if (len % 8) throw std::invalid_argument("length must be a multiple of 8");
    if ((len && !buf) || !out) throw std::invalid_argument("null buffer");
    *out = checksum_words(buf, len, base_word);
    return PAES_OK;
  });
}

int paes_cuda_checksum_device(const void* d_buf, uint64_t len, uint64_t base_word, uint64_t* out, int device_id,
                              void* stream) {
  return guarded([&] {
    if (len % 8) throw std::invalid_argument("length must be a multiple of 8");
    if (!out) throw std::invalid_argument("null output");
    if (len && (!d_buf || reinterpret_cast<std::uintptr_t>(d_buf) % 8)) throw std::invalid_argument("bad device buffer");
    DevCtx& d = device(device_id);
    DeviceGuard g(device_id);
    std::lock_guard<std::mutex> lk(d.mu);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    PAES_CK(cudaMemsetAsync(d.d_acc, 0, 8, s));
    PAES_CK(launch_checksum(d_buf, len / 8, base_word, d.d_acc, d.sm_count, s));
    PAES_CK(cudaMemcpyAsync(d.h_acc, d.d_acc, 8, cudaMemcpyDeviceToHost, s));
    PAES_CK(cudaStreamSynchronize(s));
    *out = *d.h_acc;
    return PAES_OK;
  });
}

int paes_cuda_count_mismatch_device(const void* d_a, const void* d_b, uint64_t len, uint64_t* out, int device_id,
                                    void* stream) {
  return guarded([&] {
    if (len % 16) throw std::invalid_argument("length must be a multiple of 16");
    if (!out) throw std::invalid_argument("null output");
    if (len && (!d_a || !d_b || (reinterpret_cast<std::uintptr_t>(d_a) | reinterpret_cast<std::uintptr_t>(d_b)) % 16))
      throw std::invalid_argument("device buffers must be 16-byte aligned");
    DevCtx& d = device(device_id);
    DeviceGuard g(device_id);
    std::lock_guard<std::mutex> lk(d.mu);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    PAES_CK(cudaMemsetAsync(d.d_acc, 0, 8, s));
    PAES_CK(launch_mismatch(d_a, d_b, len / 16, d.d_acc, d.sm_count, s));
    PAES_CK(cudaMemcpyAsync(d.h_acc, d.d_acc, 8, cudaMemcpyDeviceToHost, s));
    PAES_CK(cudaStreamSynchronize(s));
    *out = *d.h_acc;
    return PAES_OK;
  });
}

uint64_t paes_cuda_launch_count(void) { return launch_count(); }

}  // extern "C"

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
  const std::uint64_t step = ((n / parts) + 4095) & ~std::uint64_t(4095);
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
// back into the same slot, pwrite -- all slots in flight at once.  Returns
// the output bytes written (decrypt final: unpadded).
std::uint64_t file_shard(DevCtx& d, const Range& r, int in_fd, int out_fd, std::uint8_t* out_map, std::uint64_t off,
                         const KeyWords& kw, const std::string& in_path, const std::string& out_path,
                         unsigned io_threads) {
  DeviceGuard g(d.id);
  ensure_pipeline(d, true);
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
      if (out_map)  // page faults of a shared mapping proceed in parallel; pwrite serialises on the inode
        par_io(len, io_threads, [&](std::uint64_t o, std::uint64_t n) { std::memcpy(out_map + base + o, slot + o, n); });
      else
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
  std::uint64_t out_total = 0;
  for (std::uint64_t k = 0; k < npieces; ++k) {
    const int s = static_cast<int>(k % S);
    join_slot(s);
    const std::uint64_t poff = k * C;
    const std::uint64_t len = std::min<std::uint64_t>(C, r.in_len - poff);
    const bool last = k + 1 == npieces;
    std::uint8_t* slot = d.hbuf[s];
    par_io(len, io_threads,
           [&](std::uint64_t o, std::uint64_t n) { pread_all(in_fd, slot + o, n, off + poff + o, in_path); });
    EcbArgs a = make_args(r, d.dbuf[s], d.dbuf[s], len, last, kw, d.d_status);
    if (len) PAES_CK(cudaMemcpyAsync(d.dbuf[s], d.hbuf[s], len, cudaMemcpyHostToDevice, d.st[s]));
    if (a.check_pad) PAES_CK(cudaMemsetAsync(d.d_status, 0xff, 4, d.st[s]));
    PAES_CK(launch_ecb(r.dec, a, d.sm_count, d.st[s]));
    const std::uint64_t olen = a.nblocks * 16;
    if (olen) PAES_CK(cudaMemcpyAsync(d.hbuf[s], d.dbuf[s], olen, cudaMemcpyDeviceToHost, d.st[s]));
    if (last && a.check_pad) PAES_CK(cudaMemcpyAsync(d.h_status, d.d_status, 4, cudaMemcpyDeviceToHost, d.st[s]));
    PAES_CK(cudaEventRecord(d.ev[s], d.st[s]));
    writer[s] = std::thread(write_slot, s, off + poff, olen);
    out_total = poff + olen;
  }
  for (int s = 0; s < S; ++s) join_slot(s);
  if (r.check_pad) {
    const std::uint32_t k = *d.h_status;
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
    const auto devs = device_list(static_cast<int>(workers));
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
    if (cap && ::ftruncate(out.fd, static_cast<off_t>(cap)) == 0) {
      void* p = ::mmap(nullptr, cap, PROT_READ | PROT_WRITE, MAP_SHARED, out.fd, 0);
      if (p != MAP_FAILED) {
        map.p = static_cast<std::uint8_t*>(p);
        map.n = cap;
      }
    }
    std::vector<std::uint64_t> produced(plan.size(), 0);
    std::vector<std::string> failures(plan.size());
    auto work = [&](std::size_t i) {
      const Chunk& c = plan[i];
      Range r;
      r.dec = dec;
      r.in_len = c.raw_len;
      r.pad = !dec && c.is_final;
      r.check_pad = dec && c.is_final;
      try {
        DevCtx& d = device(devs[i]);
        std::lock_guard<std::mutex> lk(d.mu);
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        const unsigned io = g_io_threads_per_shard
                                ? g_io_threads_per_shard
                                : std::clamp<unsigned>(hw / static_cast<unsigned>(plan.size()), 1u, 8u);
        produced[i] = file_shard(d, r, in.fd, out.fd, map.p, c.offset, kw, in_path, tmp, io);
      } catch (const CudaFail& e) {
        failures[i] = e.msg;
      } catch (const IoFail& e) {
        failures[i] = e.msg;
      } catch (const std::exception& e) {
        failures[i] = e.what();
      }
    };
    if (plan.size() == 1) {
      work(0);
    } else {
      std::vector<std::thread> pool;
      for (std::size_t i = 0; i < plan.size(); ++i) pool.emplace_back(work, i);
      for (auto& t : pool) t.join();
    }
    std::ostringstream failed;
    bool any = false;
    for (std::size_t i = 0; i < failures.size(); ++i) {
      if (failures[i].empty()) continue;
      failed << (any ? "; " : "") << "chunk " << i << ": " << failures[i];
      any = true;
    }
    if (any) return fail(PAES_EWORKER, "worker failure: " + failed.str());
    std::uint64_t total = 0;
    for (auto p : produced) total += p;
    if (::ftruncate(out.fd, static_cast<off_t>(total)) != 0) return fail(PAES_EIO, "truncate failed: " + tmp);
    if (::rename(tmp.c_str(), output_path) != 0) return fail(PAES_EIO, "rename failed: " + out_path);
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

// Experimental, not in include/paes_cuda.h: the bitsliced (LOP3) encrypt
// kernel for the T-table vs bitsliced A/B (scripts/bitsliced_ab.py).
extern "C" int paes_cuda_experimental_bitsliced_ecb(const void* d_in, void* d_out, uint64_t len, const uint8_t rk[176],
                                                    int device_id, void* stream) {
  return guarded([&] {
    if (len % (16 * 1024)) throw std::invalid_argument("length must be a multiple of 16 KiB");
    DevCtx& d = device(device_id);
    DeviceGuard g(device_id);
    PAES_CK(launch_ecb_bitsliced_experiment(static_cast<const std::uint8_t*>(d_in), static_cast<std::uint8_t*>(d_out),
                                            len / 16, enc_key_words(rk), d.sm_count, static_cast<cudaStream_t>(stream)));
    return PAES_OK;
  });
}
