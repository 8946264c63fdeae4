// abi_core.cu -- C ABI (include/paes_cuda.h): diagnostics, configuration,
// host rules, the ECB / chunk transforms (host and device pointers) and the
// bench/test utilities.  Reference boundary: aes::encrypt_ecb/decrypt_ecb
// (aes.hpp:86-89), paes::encrypt_chunk/decrypt_chunk (exec.hpp:61-65).
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
    set_device_list(std::vector<int>(ids, ids + n));
    return PAES_OK;
  });
}

int paes_cuda_set_pipeline(uint64_t chunk_bytes, int streams) {
  return guarded([&] {
    if (chunk_bytes % 16 != 0) throw std::invalid_argument("chunk_bytes must be a multiple of 16");
    if (chunk_bytes && chunk_bytes < 4096) throw std::invalid_argument("chunk_bytes must be >= 4096");
    if (streams < 0 || streams > 32) throw std::invalid_argument("streams must be in [0, 32]");
    set_pipeline_config(chunk_bytes, streams);
    return PAES_OK;
  });
}

int paes_cuda_set_zero_copy_max(uint64_t bytes) {
  return guarded([&] {
    set_zero_copy_max(bytes);
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

uint32_t paes_cuda_auto_shards(uint64_t len, uint32_t ndev) { return auto_shards(len, ndev); }

int paes_cuda_sbox(int inverse, uint8_t out[256]) {
  if (!out) return fail(PAES_EINVAL, "null buffer");
  std::memcpy(out, inverse ? kTables.inv_sbox : kTables.sbox, 256);
  return PAES_OK;
}

int paes_cuda_state_transform(int op, uint8_t* states, uint64_t n, const uint8_t rk16[16]) {
  return guarded([&] {
    if (op < PAES_OP_SUB_BYTES || op > PAES_OP_ADD_ROUND_KEY) throw std::invalid_argument("bad state op");
    if (op == PAES_OP_ADD_ROUND_KEY && !rk16) throw std::invalid_argument("null round key");
    if (n == 0) return PAES_OK;
    if (!states) throw std::invalid_argument("null states");
    if (n > (1ull << 32)) throw std::invalid_argument("too many states");
    StateKey k{};
    if (op == PAES_OP_ADD_ROUND_KEY) std::memcpy(k.b, rk16, 16);
    DevCtx& d = device(device_list(1)[0]);
    DeviceGuard g(d.id);
    std::lock_guard<std::mutex> lk(d.mu);
    ensure_pipeline(d, false);
    QuiesceOnThrow quiesce{d};
    cudaStream_t s = d.st[0];
    std::uint8_t* dp = nullptr;
    PAES_CK(cudaMallocAsync(reinterpret_cast<void**>(&dp), 16 * n, s));
    PAES_CK(cudaMemcpyAsync(dp, states, 16 * n, cudaMemcpyHostToDevice, s));
    PAES_CK(launch_state_op(op, dp, n, k, s));
    PAES_CK(cudaMemcpyAsync(states, dp, 16 * n, cudaMemcpyDeviceToHost, s));
    PAES_CK(cudaFreeAsync(dp, s));
    PAES_CK(cudaStreamSynchronize(s));
    return PAES_OK;
  });
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
    check_alias(d_in, len, d_out, len);
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

}  // extern "C"

namespace {

// Argument rules of encrypt_chunk / decrypt_chunk (exec.cpp:375-392,
// chunk.cpp:90-100) for the device-pointer entries, checked on the host
// before any device work; returns the transform's range and output bytes.
Range device_chunk_range(int dir, const void* d_in, uint64_t len, int is_final, const uint8_t* rk, const void* d_out,
                         uint64_t* out_bytes) {
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
  r.in_len = len;
  *out_bytes = r.pad ? (len / 16 + 1) * 16 : len;
  if (*out_bytes && ((len && !d_in) || !d_out)) throw std::invalid_argument("null device buffer");
  check_alias(d_in, len, d_out, *out_bytes);
  return r;
}

}  // namespace

extern "C" {

int paes_cuda_chunk_device(int dir, const void* d_in, uint64_t len, int is_final, const uint8_t rk[176], void* d_out,
                           uint64_t* out_len, int device_id, void* stream) {
  return guarded([&] {
    uint64_t out_bytes = 0;
    const Range r = device_chunk_range(dir, d_in, len, is_final, rk, d_out, &out_bytes);
    if (out_bytes == 0) {
      if (out_len) *out_len = 0;
      return PAES_OK;
    }
    DevCtx& d = device(device_id);
    DeviceGuard g(device_id);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const KeyWords kw = r.dec ? dec_key_words(rk) : enc_key_words(rk);
    if (!r.check_pad) {
      EcbArgs a = make_args(r, static_cast<const std::uint8_t*>(d_in), static_cast<std::uint8_t*>(d_out), len, true,
                            kw, nullptr);
      PAES_CK(launch_ecb(r.dec, a, d.sm_count, s));
      if (out_len) *out_len = a.nblocks * 16;
      return PAES_OK;
    }
    // A final decrypt returns the unpadded length, so this entry waits for
    // its kernel; paes_cuda_chunk_device_async is the queued / graph form.
    StatusSlot slot(d);  // a status word of this call's own: concurrent decrypts do not serialise
    EcbArgs a = make_args(r, static_cast<const std::uint8_t*>(d_in), static_cast<std::uint8_t*>(d_out), len, true, kw,
                          slot.dev());
    // the trailer check writes the mapped word itself: no memset / D2H copy
    *reinterpret_cast<volatile std::uint32_t*>(slot.host()) = 0xffffffffu;  // sentinel: unchecked => PaddingError
    PAES_CK(launch_ecb(true, a, d.sm_count, s));
    PAES_CK(cudaStreamSynchronize(s));
    const std::uint32_t k = *reinterpret_cast<volatile std::uint32_t*>(slot.host());
    if (k == 0xffffffffu) throw PaddingError("unpad: invalid pad bytes");
    if (out_len) *out_len = len - k;
    return PAES_OK;
  });
}

int paes_cuda_chunk_device_async(int dir, const void* d_in, uint64_t len, int is_final, const uint8_t rk[176],
                                 void* d_out, uint64_t* d_result, int device_id, void* stream) {
  return guarded([&] {
    if (!d_result || reinterpret_cast<std::uintptr_t>(d_result) % 8)
      throw std::invalid_argument("d_result must be an 8-byte aligned device-visible word");
    uint64_t out_bytes = 0;
    const Range r = device_chunk_range(dir, d_in, len, is_final, rk, d_out, &out_bytes);
    DevCtx& d = device(device_id);
    DeviceGuard g(device_id);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    auto* res = reinterpret_cast<unsigned long long*>(d_result);
    if (out_bytes == 0) {  // nothing to transform: the result word still gets its value, in stream order
      PAES_CK(launch_put_u64(res, 0, s));
      return PAES_OK;
    }
    EcbArgs a = make_args(r, static_cast<const std::uint8_t*>(d_in), static_cast<std::uint8_t*>(d_out), len, true,
                          r.dec ? dec_key_words(rk) : enc_key_words(rk), nullptr);
    a.result = res;
    PAES_CK(launch_ecb(r.dec, a, d.sm_count, s));
    return PAES_OK;
  });
}

}  // extern "C"

extern "C" {

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
