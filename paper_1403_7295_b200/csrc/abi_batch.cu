// abi_batch.cu -- C ABI of the multi-key batch path (config 5): one-shot
// device batches, prepared plans, and the pipelined host-pointer batch.
// Replaces per-message encrypt_chunk loops (exec.cpp:375-392).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "runtime.hpp"

using namespace paes_b200;
using namespace paes_b200::rt;

// ------------------------------------------------------------ batch (config 5)
namespace {

// Host image of a batch: BatchMsg[n] | KeyWords[n] (| status words when the
// trailers are checked).  Validation mirrors encrypt_chunk / decrypt_chunk per
// message (exec.cpp:375-392).
struct BatchImage {
  bool dec = false, check = false;
  bool aligned = true;  // every in/out offset a multiple of 16
  std::uint32_t n = 0;
  unsigned long long total_tiles = 0;  // warp tiles (each message owns whole tiles)
  std::size_t msg_bytes = 0, keys_off = 0, image_bytes = 0, status_off = 0, total_bytes = 0;
  bool has_empty = false;  // some message has no output block (its length is written by the host)
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
    if (in_off[i] % 16 || out_off[i] % 16) b.aligned = false;  // any byte offset works; aligned ones are faster
    if ((b.dec || !pad) && lens[i] % 16) throw std::invalid_argument("message length must be a multiple of 16");
    if (b.check && lens[i] == 0) throw PaddingError("unpad: length must be a non-zero multiple of 16");
    const unsigned long long nb = lens[i] / 16 + ((pad && !b.dec) ? 1 : 0);
    if (nb > 0xffffffffull) throw std::invalid_argument("message too large for the batch path");
    if (lens[i] > UINT64_MAX - in_off[i] || 16 * nb > UINT64_MAX - out_off[i])
      throw std::invalid_argument("batch message span overflows the address range");
    b.nblocks[i] = static_cast<std::uint32_t>(nb);
    if (nb == 0) b.has_empty = true;
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
  a.aligned = b.aligned ? 1u : 0u;
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
  // the previous upload (on whichever device) must finish reading the buffer
  if (st.ev) PAES_CK(cudaEventSynchronize(st.ev));
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

// Per-thread device image for one-shot batches, reused call to call.  A
// stream-ordered malloc/free per call let the pool trim at every sync point,
// and some calls then took twice as long (scripts/oneshot_batch_probe.py).
// Reuse is guarded by an event recorded after the kernel that read the image:
// the next call's upload waits on it in stream order.
struct DevImage {
  int device = -1;
  std::uint8_t* p = nullptr;
  std::size_t cap = 0;
  cudaEvent_t done = nullptr;
  void release() {
    if (done) {
      cudaEventSynchronize(done);
      cudaEventDestroy(done);
    }
    if (p) {
      int prev = -1;
      cudaGetDevice(&prev);
      cudaSetDevice(device);
      cudaFree(p);
      if (prev >= 0) cudaSetDevice(prev);
    }
    p = nullptr, cap = 0, done = nullptr;
  }
  ~DevImage() { release(); }
};
thread_local DevImage t_dimg;

std::uint8_t* device_image(std::size_t bytes, int device, cudaStream_t s) {
  DevImage& di = t_dimg;
  if (di.device != device) {
    di.release();
    di.device = device;
  }
  if (!di.done) PAES_CK(cudaEventCreateWithFlags(&di.done, cudaEventDisableTiming));
  if (di.cap < bytes) {
    PAES_CK(cudaEventSynchronize(di.done));
    if (di.p) PAES_CK(cudaFree(di.p));
    di.p = nullptr;
    di.cap = 0;
    PAES_CK(cudaMalloc(reinterpret_cast<void**>(&di.p), bytes));
    di.cap = bytes;
  }
  PAES_CK(cudaStreamWaitEvent(s, di.done, 0));  // the previous call's kernel has finished reading it
  return di.p;
}

}  // namespace

struct paes_batch_plan {
  int device = -1;
  BatchImage img;
  std::uint8_t* dd = nullptr;        // device image
  std::uint32_t* h_status = nullptr;  // pinned
  std::mutex check_mu;  // checked runs share the status words: one at a time
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
    std::uint8_t* dd = device_image(b.total_bytes, device_id, s);
    PAES_CK(cudaMemcpyAsync(dd, host, b.image_bytes, cudaMemcpyHostToDevice, s));
    PAES_CK(cudaEventRecord(t_stage.ev, s));
    PAES_CK(launch_batch(b.dec, batch_args(b, d_in, d_out, dd), d.sm_count, s));
    if (b.check) {
      auto* st = reinterpret_cast<std::uint32_t*>(host + b.status_off);
      PAES_CK(cudaMemcpyAsync(st, dd + b.status_off, 4ull * n, cudaMemcpyDeviceToHost, s));
      PAES_CK(cudaEventRecord(t_dimg.done, s));
      PAES_CK(cudaStreamSynchronize(s));
      finish_lengths(b, st, out_lens);
    } else {
      PAES_CK(cudaEventRecord(t_dimg.done, s));
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
    if (!b.check) {  // descriptors are read-only: unchecked runs may overlap freely
      PAES_CK(launch_batch(b.dec, batch_args(b, d_in, d_out, plan->dd), d.sm_count, s));
      finish_lengths(b, nullptr, out_lens);
      return PAES_OK;
    }
    std::lock_guard<std::mutex> lk(plan->check_mu);
    PAES_CK(launch_batch(b.dec, batch_args(b, d_in, d_out, plan->dd), d.sm_count, s));
    PAES_CK(cudaMemcpyAsync(plan->h_status, plan->dd + b.status_off, 4ull * b.n, cudaMemcpyDeviceToHost, s));
    PAES_CK(cudaStreamSynchronize(s));
    finish_lengths(b, plan->h_status, out_lens);
    return PAES_OK;
  });
}

int paes_cuda_batch_plan_run_async(paes_batch_plan* plan, const void* d_in, void* d_out, uint64_t* d_out_lens,
                                   void* stream) {
  return guarded([&] {
    if (!plan) throw std::invalid_argument("null plan");
    if (!d_out_lens || reinterpret_cast<std::uintptr_t>(d_out_lens) % 8)
      throw std::invalid_argument("d_out_lens must be an 8-byte aligned device-visible array");
    const BatchImage& b = plan->img;
    if (b.n == 0) return PAES_OK;
    if (!d_in || !d_out) throw std::invalid_argument("null device buffer");
    DevCtx& d = device(plan->device);
    DeviceGuard dg(plan->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // messages without an output block own no tile, so no thread writes them
    if (b.has_empty) PAES_CK(cudaMemsetAsync(d_out_lens, 0, 8ull * b.n, s));
    BatchArgs a = batch_args(b, d_in, d_out, plan->dd);
    a.status = nullptr;  // the verdicts go to the caller's array: runs never share state
    a.out_lens = reinterpret_cast<unsigned long long*>(d_out_lens);
    PAES_CK(launch_batch(b.dec, a, d.sm_count, s));
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
    QuiesceOnThrow quiesce{d};
    const std::uint64_t cap = d.chunk;  // ring slot capacity
    const int S = static_cast<int>(d.st.size());
    // group target: the ring's piece-size model over the batch's input bytes
    std::uint64_t in_bytes = 0;
    for (std::uint32_t i = 0; i < n; ++i) in_bytes += lens[i];
    const std::uint64_t C = piece_size(in_bytes, cap, S);
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
    // persistent buffers: per-stream output spans (obuf; the input spans use
    // the ring's dbuf) and ONE device image holding every group's
    // descriptors, uploaded by a single copy before the groups start (a
    // small copy per group queued behind each input span cost ~8 % of the
    // PCIe rate, scripts/batch_host_probe.py).  Stream-ordered allocations
    // per group would let the pool serialise groups across streams.
    if (static_cast<int>(d.obuf.size()) != S) {  // all or nothing: a partial ring must not survive a failure
      for (auto p : d.obuf) cudaFree(p);
      d.obuf.clear();
      try {
        for (int i = 0; i < S; ++i) {
          std::uint8_t* p = nullptr;
          PAES_CK(cudaMalloc(&p, cap + 16));
          d.obuf.push_back(p);
        }
      } catch (...) {
        for (auto p : d.obuf) cudaFree(p);
        d.obuf.clear();
        throw;
      }
    }
    if (d.dsc.empty()) {
      d.dsc.push_back(nullptr);
      d.dsc_cap.push_back(0);
    }
    if (d.dsc_cap[0] < total) {
      for (auto st : d.st) PAES_CK(cudaStreamSynchronize(st));
      if (d.dsc[0]) PAES_CK(cudaFree(d.dsc[0]));
      d.dsc[0] = nullptr;
      d.dsc_cap[0] = 0;
      PAES_CK(cudaMalloc(&d.dsc[0], total));
      d.dsc_cap[0] = total;
    }
    std::uint8_t* const dimg = d.dsc[0];
    // one queue per engine, as the pinned ring (runtime.cu run_host_range):
    // copy-in on st[0], kernels on st[1], copy-out on st[2], per-slot events.
    // Group k+S's copy-in reuses dbuf[slot] once group k's kernel has read
    // it; its kernel reuses obuf[slot] once group k's copy-out is done.
    cudaStream_t sin = d.st[0], sk = d.st[1 % S], sout = d.st[2 % S];
    PAES_CK(cudaMemcpyAsync(dimg, host, total, cudaMemcpyHostToDevice, sin));  // ordered before every ev_in
    for (std::size_t k = 0; k < groups.size(); ++k) {
      const Group& g = groups[k];
      const BatchImage& b = imgs[k];
      const int slot = static_cast<int>(k % S);
      const bool reuse = k >= static_cast<std::size_t>(S);
      const bool fits = g.in_hi - g.in_lo <= cap + 16 && g.out_hi - g.out_lo <= cap + 16;
      std::uint8_t* din = d.dbuf[slot];
      std::uint8_t* dout = d.obuf[slot];
      std::uint8_t* dd = dimg + img_off[k];
      if (reuse) PAES_CK(cudaStreamWaitEvent(sin, d.ev_k[slot], 0));
      if (!fits) {  // a single message larger than the staging chunk
        PAES_CK(cudaMallocAsync(reinterpret_cast<void**>(&din), std::max<std::uint64_t>(16, g.in_hi - g.in_lo), sin));
        PAES_CK(cudaMallocAsync(reinterpret_cast<void**>(&dout), std::max<std::uint64_t>(16, g.out_hi - g.out_lo), sin));
      }
      if (g.in_hi > g.in_lo) PAES_CK(copy_h2d_aligned(din, h_in + g.in_lo, g.in_hi - g.in_lo, sin));
      PAES_CK(cudaEventRecord(d.ev_in[slot], sin));
      PAES_CK(cudaStreamWaitEvent(sk, d.ev_in[slot], 0));
      if (reuse) PAES_CK(cudaStreamWaitEvent(sk, d.ev_out[slot], 0));
      PAES_CK(launch_batch(b.dec, batch_args(b, din, dout, dd), d.sm_count, sk));
      PAES_CK(cudaEventRecord(d.ev_k[slot], sk));
      PAES_CK(cudaStreamWaitEvent(sout, d.ev_k[slot], 0));
      // copy back only the messages' output bytes, merged where they touch:
      // gaps between messages in h_out belong to the caller and are never
      // written (a packed layout such as config 5 is still one copy per group)
      std::vector<std::pair<std::uint64_t, std::uint64_t>> rs;
      rs.reserve(g.count);
      for (std::uint32_t i = g.first; i < g.first + g.count; ++i)
        if (all.nblocks[i]) rs.emplace_back(out_off[i], out_off[i] + 16ull * all.nblocks[i]);
      std::sort(rs.begin(), rs.end());
      for (std::size_t r = 0; r < rs.size();) {
        std::uint64_t lo = rs[r].first, hi = rs[r].second;
        for (++r; r < rs.size() && rs[r].first <= hi; ++r) hi = std::max(hi, rs[r].second);
        PAES_CK(copy_d2h_aligned(h_out + lo, dout + (lo - g.out_lo), hi - lo, sout));
      }
      if (b.check)
        PAES_CK(cudaMemcpyAsync(host + img_off[k] + b.status_off, dd + b.status_off, 4ull * b.n,
                                cudaMemcpyDeviceToHost, sout));
      if (!fits) {
        PAES_CK(cudaFreeAsync(din, sout));
        PAES_CK(cudaFreeAsync(dout, sout));
      }
      PAES_CK(cudaEventRecord(d.ev_out[slot], sout));
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

}  // extern "C"
