// aes_bitsliced.cu -- bitsliced AES-128 ECB encrypt for sm_100a: the ALU
// (LOP3) alternative the north_star asks to A/B against the T-table kernel.
// Not on the product path and not in libpaes_cuda.so: build.py links it into
// its own A/B library, lib/libpaes_bitsliced_ab.so, whose only entry point
// paes_bitsliced_ab_ecb is used by scripts/bitsliced_ab.py and
// tests/test_gpu_bitsliced.py.
//
// Layout: each thread owns 32 blocks of a 1024-block warp tile (lane l takes
// blocks l, l+32, ..., so every 128-bit load/store is coalesced).  The 32x4
// column words are transposed into 128 bit-planes p[c][b] (bit j of
// p[c][b] = bit b of column word c of block j), with PRMT for the 16- and
// 8-bit levels of the 32x32 transpose and SWAPMOVE for the rest.  A round is
// then 16 bitsliced S-box circuits (generated, verified: sbox_bitsliced.inc),
// ShiftRows as register renaming, and MixColumns fused with AddRoundKey,
// whose key bits come in as all-zero/all-one masks from the kernel parameter
// constant bank (uniform operands of LOP3).
#include <cuda_runtime.h>

#include <cstdint>

#include "aes_kernels.cuh"
#include "host_rules.hpp"

namespace paes_b200 {

namespace {

#include "sbox_bitsliced.inc"

struct BsKeys {
  std::uint32_t m[11][4][32];  // m[r][c][b] = bit b of round key r, column word c ? ~0u : 0u
};

constexpr int kBsThreads = 128;

// In-place LSB-first 32x32 bit transpose of a[0..31] (a[k] bit i <-> a[i] bit k).
__device__ __forceinline__ void transpose32(std::uint32_t (&a)[32]) {
  // j = 16: swap halfwords between rows k and k+16
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const std::uint32_t x = a[k], y = a[k + 16];
    a[k] = __byte_perm(x, y, 0x5410);       // [x.lo16, y.lo16]
    a[k + 16] = __byte_perm(x, y, 0x7632);  // [x.hi16, y.hi16]
  }
  // j = 8: swap bytes between rows k and k+8
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    if (k & 8) continue;
    const std::uint32_t x = a[k], y = a[k + 8];
    a[k] = __byte_perm(x, y, 0x6240);      // [x.b0, y.b0, x.b2, y.b2]
    a[k + 8] = __byte_perm(x, y, 0x7351);  // [x.b1, y.b1, x.b3, y.b3]
  }
  // j = 4, 2, 1: SWAPMOVE
#pragma unroll
  for (int j = 4, s = 0; j > 0; j >>= 1, ++s) {
    const std::uint32_t m = s == 0 ? 0x0F0F0F0Fu : s == 1 ? 0x33333333u : 0x55555555u;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      if (k & j) continue;
      const std::uint32_t t = ((a[k] >> j) ^ a[k + j]) & m;
      a[k] ^= t << j;
      a[k + j] ^= t;
    }
  }
}

__device__ __forceinline__ void sbox8(std::uint32_t* x) { sbox_bitsliced(x[0], x[1], x[2], x[3], x[4], x[5], x[6], x[7]); }

// p[c][8r + i]: bit i of byte (row r, column c) for the thread's 32 blocks.
__global__ void __launch_bounds__(kBsThreads) ecb_bitsliced_kernel(const std::uint8_t* in, std::uint8_t* out,
                                                                   unsigned long long ntiles,
                                                                   const __grid_constant__ BsKeys k) {
  const std::uint32_t lane = threadIdx.x & 31;
  const unsigned long long wpc = blockDim.x / 32;
  for (unsigned long long tile = blockIdx.x * wpc + threadIdx.x / 32; tile < ntiles; tile += gridDim.x * wpc) {
    const unsigned long long base = tile * 1024ull + lane;
    std::uint32_t p[4][32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const uint4 v = __ldcs(reinterpret_cast<const uint4*>(in + 16ull * (base + 32ull * j)));
      p[0][j] = v.x;
      p[1][j] = v.y;
      p[2][j] = v.z;
      p[3][j] = v.w;
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) transpose32(p[c]);
    // round 0: AddRoundKey
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int b = 0; b < 32; ++b) p[c][b] ^= k.m[0][c][b];
    // rounds 1..9: SubBytes, ShiftRows, MixColumns + AddRoundKey
#pragma unroll 1
    for (int r = 1; r < 10; ++r) {
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int row = 0; row < 4; ++row) sbox8(&p[c][8 * row]);
      std::uint32_t q[4][32];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        // shifted column: a_row = byte (row, c + row)
        const std::uint32_t* a0 = &p[c][0];
        const std::uint32_t* a1 = &p[(c + 1) & 3][8];
        const std::uint32_t* a2 = &p[(c + 2) & 3][16];
        const std::uint32_t* a3 = &p[(c + 3) & 3][24];
        const std::uint32_t* a[4] = {a0, a1, a2, a3};
#pragma unroll
        for (int row = 0; row < 4; ++row) {
          const std::uint32_t* x = a[row];
          const std::uint32_t* y = a[(row + 1) & 3];
          const std::uint32_t* z = a[(row + 2) & 3];
          const std::uint32_t* w = a[(row + 3) & 3];
          std::uint32_t t[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) t[i] = x[i] ^ y[i];  // t = a_row ^ a_row+1
          // xtime(t) ^ a_row+1 ^ a_row+2 ^ a_row+3 ^ key
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            std::uint32_t xt = i == 0 ? t[7] : t[i - 1];
            if (i == 1 || i == 3 || i == 4) xt ^= t[7];
            q[c][8 * row + i] = xt ^ y[i] ^ z[i] ^ w[i] ^ k.m[r][c][8 * row + i];
          }
        }
      }
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int b = 0; b < 32; ++b) p[c][b] = q[c][b];
    }
    // round 10: SubBytes, ShiftRows, AddRoundKey
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int row = 0; row < 4; ++row) sbox8(&p[c][8 * row]);
    std::uint32_t q[4][32];
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int row = 0; row < 4; ++row)
#pragma unroll
        for (int i = 0; i < 8; ++i) q[c][8 * row + i] = p[(c + row) & 3][8 * row + i] ^ k.m[10][c][8 * row + i];
#pragma unroll
    for (int c = 0; c < 4; ++c) transpose32(q[c]);
#pragma unroll
    for (int j = 0; j < 32; ++j)
      __stcs(reinterpret_cast<uint4*>(out + 16ull * (base + 32ull * j)), make_uint4(q[0][j], q[1][j], q[2][j], q[3][j]));
  }
}

}  // namespace

// Whole 1024-block tiles only (the A/B driver sizes its buffers accordingly).
static cudaError_t launch_bitsliced(const std::uint8_t* in, std::uint8_t* out, unsigned long long nblocks,
                                    const KeyWords& kw, cudaStream_t stream) {
  if (nblocks % 1024) return cudaErrorInvalidValue;
  BsKeys k{};
  for (int r = 0; r < 11; ++r)
    for (int c = 0; c < 4; ++c)
      for (int b = 0; b < 32; ++b) k.m[r][c][b] = ((kw.w[4 * r + c] >> b) & 1u) ? 0xffffffffu : 0u;
  int dev = 0, sm_count = 0, per_sm = 0;
  cudaError_t e;
  if ((e = cudaGetDevice(&dev)) || (e = cudaDeviceGetAttribute(&sm_count, cudaDevAttrMultiProcessorCount, dev)) ||
      (e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ecb_bitsliced_kernel, kBsThreads, 0)))
    return e;
  const unsigned long long ntiles = nblocks / 1024;
  unsigned long long grid = (ntiles + kBsThreads / 32 - 1) / (kBsThreads / 32);
  const unsigned long long cap = static_cast<unsigned long long>(sm_count) * (per_sm > 0 ? per_sm : 1);
  if (grid > cap) grid = cap;
  if (grid == 0) return cudaSuccess;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(kBsThreads);
  cfg.stream = stream;
  return cudaLaunchKernelEx(&cfg, ecb_bitsliced_kernel, in, out, ntiles, k);
}

}  // namespace paes_b200

// The A/B library's one entry point (current device; 0 ok, -22 for a length
// that is not whole 16 KiB tiles, -1002 for a CUDA error).
extern "C" int paes_bitsliced_ab_ecb(const void* d_in, void* d_out, std::uint64_t len, const std::uint8_t rk[176],
                                     void* stream) {
  if (len % (16 * 1024) || !rk) return -22;
  const cudaError_t e =
      paes_b200::launch_bitsliced(static_cast<const std::uint8_t*>(d_in), static_cast<std::uint8_t*>(d_out), len / 16,
                                  paes_b200::enc_key_words(rk), static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? 0 : -1002;
}
