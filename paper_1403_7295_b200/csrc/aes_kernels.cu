// aes_kernels.cu -- sm_100a kernels + their host launch wrappers.
// See aes_kernels.cuh for the design; DESIGN.md for the roofline.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <utility>

#include "../../include/paes_cuda.h"
#include "aes_kernels.cuh"
#include "launch.hpp"

namespace paes_b200 {

// Generated tables, constant-initialised from the constexpr host build.
__device__ const AesTables g_tab = kTables;

std::atomic<unsigned long long> g_launches{0};

namespace {

// Programmatic dependent launch for ecb_kernel (PAES_PDL=0 builds plain
// launches): measured on queued C launches (scripts/mid_launch_probe.cu,
// profiles/r01_pdl_ab.json) 16 MiB 703 -> 786 GB/s, 64 MiB 819 -> 848,
// 1 GiB 869 -> 870; a single launch loses the first-tile prefetch that used
// to hide behind the table staging (0-2 %).
#ifndef PAES_PDL
#define PAES_PDL 1
#endif
#ifndef PAES_PREFETCH
#define PAES_PREFETCH 1  // tiles per warp prefetched into L2 before griddepcontrol.wait (0 = off)
#endif
#ifndef PAES_THREADS
#define PAES_THREADS 512
#endif
constexpr int kThreads = PAES_THREADS;  // one persistent CTA per SM (smem-limited)

// ---------------------------------------------------------------- staging
// Replicate the tables 32x (one copy per bank) into the CTA's shared memory.
// word index w:  region = w >> 14, row x = (w >> 6) & 255, table-in-region
// t = (w >> 5) & 1, lane = w & 31.  Four consecutive words (4 lanes) share a
// value, so the fill is one 16-byte store per 4 words.
// Two phases: the CTA first copies the 1 KiB base table (+ InvS) into a
// scratch area with a handful of coalesced loads, then every thread expands
// its share from that copy (broadcast LDS, 2 rows per warp per pass).  Reading
// the base table straight from global memory in the fill put every thread of
// all 148 SMs on the same few L2 lines: ~2-3 us of contention per launch
// (profiles/r01_small_latency.json: staging 4.1 us with 1 CTA, 6-7 with 148).
// The trip count is a compile-time constant (kernels launch with kThreads), so
// the fill loop unrolls.
template <bool DEC>
__device__ __forceinline__ void stage_tables(std::uint32_t* sm) {
  constexpr int kTabBytes = DEC ? kDecSmemBytes : kEncSmemBytes;
  constexpr int nvec = kTabBytes / 16;
  static_assert(nvec % kThreads == 0, "staging assumes whole passes");
  // the CTA's single copy of the base table (+ InvS): 8-10 coalesced requests
  std::uint32_t* base = sm + kTabBytes / 4;
  constexpr int kScratchWords = 256 + (DEC ? 64 : 0);
#pragma unroll
  for (int w = static_cast<int>(threadIdx.x); w < kScratchWords; w += kThreads)
    base[w] = w < 256 ? (DEC ? g_tab.td0 : g_tab.te0)[w]
                      : reinterpret_cast<const std::uint32_t*>(g_tab.inv_sbox)[w - 256];
  __syncthreads();
  const std::uint8_t* inv_sbox = reinterpret_cast<const std::uint8_t*>(base + 256);
#pragma unroll
  for (int it = 0; it < nvec / kThreads; ++it) {
    const int i = it * kThreads + static_cast<int>(threadIdx.x);
    const int w = i * 4;
    const int region = w >> 14;
    const int x = (w >> 6) & 255;
    const int t = (w >> 5) & 1;
    std::uint32_t v;
    if (region < 2) {
      v = base[x];
      const int rot = (region * 2 + t) * 8;
      v = (v << rot) | (rot ? (v >> (32 - rot)) : 0u);
    } else {
      v = t == 0 ? static_cast<std::uint32_t>(inv_sbox[x]) * 0x01010101u : 0u;
    }
    reinterpret_cast<uint4*>(sm)[i] = make_uint4(v, v, v, v);
  }
}

// ---------------------------------------------------------------- lookups
// (byte_k(w) << 8) | lane*4  -- one PRMT; the table offset is the LDS immediate.
#define PAES_PERM(w, k) __byte_perm((w), lane4, 0x5504 | ((k) << 4))
#define PAES_TL(w, k, OFF) (*reinterpret_cast<const std::uint32_t*>(smb + PAES_PERM(w, k) + (OFF)))

// bytes {a.b0, b.b1, c.b2, d.b3}
__device__ __forceinline__ std::uint32_t pick4(std::uint32_t a, std::uint32_t b, std::uint32_t c, std::uint32_t d) {
  const std::uint32_t p = __byte_perm(a, b, 0x7650);
  const std::uint32_t q = __byte_perm(c, d, 0x7210);
  return __byte_perm(p, q, 0x7610);
}

struct Block4 {
  std::uint32_t x, y, z, w;
};

// One encrypt T-round on NB blocks (round key words kw[4r..4r+3]).
template <int NB, class K>
__device__ __forceinline__ void enc_round(Block4 (&s)[NB], const K& kw, int r, const char* smb, std::uint32_t lane4) {
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    const std::uint32_t s0 = s[j].x, s1 = s[j].y, s2 = s[j].z, s3 = s[j].w;
    s[j].x = PAES_TL(s0, 0, kT0) ^ PAES_TL(s1, 1, kT1) ^ PAES_TL(s2, 2, kT2) ^ PAES_TL(s3, 3, kT3) ^ kw[4 * r + 0];
    s[j].y = PAES_TL(s1, 0, kT0) ^ PAES_TL(s2, 1, kT1) ^ PAES_TL(s3, 2, kT2) ^ PAES_TL(s0, 3, kT3) ^ kw[4 * r + 1];
    s[j].z = PAES_TL(s2, 0, kT0) ^ PAES_TL(s3, 1, kT1) ^ PAES_TL(s0, 2, kT2) ^ PAES_TL(s1, 3, kT3) ^ kw[4 * r + 2];
    s[j].w = PAES_TL(s3, 0, kT0) ^ PAES_TL(s0, 1, kT1) ^ PAES_TL(s1, 2, kT2) ^ PAES_TL(s2, 3, kT3) ^ kw[4 * r + 3];
  }
}

// Last encrypt round: S[x] sits at byte r of Te_{(r+3)%4}[x].
template <int NB, class K>
__device__ __forceinline__ void enc_last(Block4 (&s)[NB], const K& kw, const char* smb, std::uint32_t lane4) {
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    const std::uint32_t s0 = s[j].x, s1 = s[j].y, s2 = s[j].z, s3 = s[j].w;
    s[j].x = pick4(PAES_TL(s0, 0, kT3), PAES_TL(s1, 1, kT0), PAES_TL(s2, 2, kT1), PAES_TL(s3, 3, kT2)) ^ kw[40];
    s[j].y = pick4(PAES_TL(s1, 0, kT3), PAES_TL(s2, 1, kT0), PAES_TL(s3, 2, kT1), PAES_TL(s0, 3, kT2)) ^ kw[41];
    s[j].z = pick4(PAES_TL(s2, 0, kT3), PAES_TL(s3, 1, kT0), PAES_TL(s0, 2, kT1), PAES_TL(s1, 3, kT2)) ^ kw[42];
    s[j].w = pick4(PAES_TL(s3, 0, kT3), PAES_TL(s0, 1, kT0), PAES_TL(s1, 2, kT1), PAES_TL(s2, 3, kT2)) ^ kw[43];
  }
}

// Equivalent inverse cipher round (InvShiftRows: column j row r <- column j-r).
template <int NB, class K>
__device__ __forceinline__ void dec_round(Block4 (&s)[NB], const K& kw, int r, const char* smb, std::uint32_t lane4) {
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    const std::uint32_t s0 = s[j].x, s1 = s[j].y, s2 = s[j].z, s3 = s[j].w;
    s[j].x = PAES_TL(s0, 0, kT0) ^ PAES_TL(s3, 1, kT1) ^ PAES_TL(s2, 2, kT2) ^ PAES_TL(s1, 3, kT3) ^ kw[4 * r + 0];
    s[j].y = PAES_TL(s1, 0, kT0) ^ PAES_TL(s0, 1, kT1) ^ PAES_TL(s3, 2, kT2) ^ PAES_TL(s2, 3, kT3) ^ kw[4 * r + 1];
    s[j].z = PAES_TL(s2, 0, kT0) ^ PAES_TL(s1, 1, kT1) ^ PAES_TL(s0, 2, kT2) ^ PAES_TL(s3, 3, kT3) ^ kw[4 * r + 2];
    s[j].w = PAES_TL(s3, 0, kT0) ^ PAES_TL(s2, 1, kT1) ^ PAES_TL(s1, 2, kT2) ^ PAES_TL(s0, 3, kT3) ^ kw[4 * r + 3];
  }
}

template <int NB, class K>
__device__ __forceinline__ void dec_last(Block4 (&s)[NB], const K& kw, const char* smb, std::uint32_t lane4) {
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    const std::uint32_t s0 = s[j].x, s1 = s[j].y, s2 = s[j].z, s3 = s[j].w;
    s[j].x = pick4(PAES_TL(s0, 0, kTS), PAES_TL(s3, 1, kTS), PAES_TL(s2, 2, kTS), PAES_TL(s1, 3, kTS)) ^ kw[40];
    s[j].y = pick4(PAES_TL(s1, 0, kTS), PAES_TL(s0, 1, kTS), PAES_TL(s3, 2, kTS), PAES_TL(s2, 3, kTS)) ^ kw[41];
    s[j].z = pick4(PAES_TL(s2, 0, kTS), PAES_TL(s1, 1, kTS), PAES_TL(s0, 2, kTS), PAES_TL(s3, 3, kTS)) ^ kw[42];
    s[j].w = pick4(PAES_TL(s3, 0, kTS), PAES_TL(s2, 1, kTS), PAES_TL(s1, 2, kTS), PAES_TL(s0, 3, kTS)) ^ kw[43];
  }
}

template <bool DEC, int NB, class K>
__device__ __forceinline__ void cipher(Block4 (&s)[NB], const K& kw, const char* smb, std::uint32_t lane4) {
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    s[j].x ^= kw[0];
    s[j].y ^= kw[1];
    s[j].z ^= kw[2];
    s[j].w ^= kw[3];
  }
#pragma unroll
  for (int r = 1; r < 10; ++r) {
    if (DEC) dec_round<NB>(s, kw, r, smb, lane4);
    else enc_round<NB>(s, kw, r, smb, lane4);
  }
  if (DEC) dec_last<NB>(s, kw, smb, lane4);
  else enc_last<NB>(s, kw, smb, lane4);
}

// ---------------------------------------------------------------- global I/O
// 16 bytes starting `sh` (0..15) bytes into the 32-byte concatenation lo:hi
// (warp-uniform switch on the word offset, then a funnel shift).
__device__ __forceinline__ Block4 bytes_at(const Block4& lo, const Block4& hi, unsigned sh) {
  const unsigned bs = (sh & 3) * 8;
  std::uint32_t w0, w1, w2, w3, w4;
  switch (sh >> 2) {
    case 0: w0 = lo.x, w1 = lo.y, w2 = lo.z, w3 = lo.w, w4 = hi.x; break;
    case 1: w0 = lo.y, w1 = lo.z, w2 = lo.w, w3 = hi.x, w4 = hi.y; break;
    case 2: w0 = lo.z, w1 = lo.w, w2 = hi.x, w3 = hi.y, w4 = hi.z; break;
    default: w0 = lo.w, w1 = hi.x, w2 = hi.y, w3 = hi.z, w4 = hi.w; break;
  }
  return Block4{__funnelshift_r(w0, w1, bs), __funnelshift_r(w1, w2, bs), __funnelshift_r(w2, w3, bs),
                __funnelshift_r(w3, w4, bs)};
}

template <bool ALIGNED>
__device__ __forceinline__ Block4 load_block(const std::uint8_t* p) {
  if (ALIGNED) {
    const uint4 v = __ldcs(reinterpret_cast<const uint4*>(p));
    return Block4{v.x, v.y, v.z, v.w};
  } else {
    // Any misalignment: the two aligned 16-byte chunks the block straddles
    // (an aligned chunk never crosses a page, so the extra bytes cannot
    // fault), then a funnel shift by the byte offset.  Every block of a
    // buffer shares the offset, so the switch is warp-uniform.  2 x LDG.128
    // per block instead of 16 byte loads: ~8x fewer L1 wavefronts.
    const std::uintptr_t a = reinterpret_cast<std::uintptr_t>(p);
    const unsigned sh = static_cast<unsigned>(a & 15);
    const uint4* q = reinterpret_cast<const uint4*>(a - sh);
    const uint4 v0 = __ldcs(q);
    if (sh == 0) return Block4{v0.x, v0.y, v0.z, v0.w};
    const uint4 v1 = __ldcs(q + 1);
    return bytes_at(Block4{v0.x, v0.y, v0.z, v0.w}, Block4{v1.x, v1.y, v1.z, v1.w}, sh);
  }
}

template <bool ALIGNED>
__device__ __forceinline__ void store_block(std::uint8_t* p, const Block4& b) {
  if (ALIGNED) {
    __stcs(reinterpret_cast<uint4*>(p), make_uint4(b.x, b.y, b.z, b.w));
  } else if ((reinterpret_cast<std::uintptr_t>(p) & 3) == 0) {  // 4-byte aligned: word stores (warp-uniform)
    std::uint32_t* q = reinterpret_cast<std::uint32_t*>(p);
    __stcs(q, b.x);
    __stcs(q + 1, b.y);
    __stcs(q + 2, b.z);
    __stcs(q + 3, b.w);
  } else {
    const std::uint32_t w[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
    for (int c = 0; c < 16; ++c) p[c] = static_cast<std::uint8_t>(w[c >> 2] >> (8 * (c & 3)));
  }
}

// A full warp row (32 consecutive blocks, lane l's at row + 16 l) stored at an
// address that is not 4-byte aligned: lane l writes the aligned 16-byte chunk
// l+1 from its own tail and lane l+1's head (one shuffle per word), lanes 0
// and 31 write the two partial end chunks byte by byte.  Every write covers
// only this row's bytes, so in-place operation and neighbouring rows are safe.
// 1 STG.128 + 4 SHFL per lane instead of 16 byte stores.
__device__ __forceinline__ void store_row_unaligned(std::uint8_t* row, const Block4& v, std::uint32_t lane) {
  const std::uintptr_t a = reinterpret_cast<std::uintptr_t>(row);
  const unsigned m = static_cast<unsigned>(a & 15);  // 1..15
  std::uint8_t* c = reinterpret_cast<std::uint8_t*>(a - m);
  const Block4 n{__shfl_down_sync(0xffffffffu, v.x, 1), __shfl_down_sync(0xffffffffu, v.y, 1),
                 __shfl_down_sync(0xffffffffu, v.z, 1), __shfl_down_sync(0xffffffffu, v.w, 1)};
  if (lane < 31) {
    const Block4 k = bytes_at(v, n, 16 - m);
    __stcs(reinterpret_cast<uint4*>(c + 16ull * (lane + 1)), make_uint4(k.x, k.y, k.z, k.w));
  }
  // the two partial end chunks, one byte per lane: lanes 0..15-m write chunk
  // 0's bytes m..15 from lane 0's block, lanes 16..15+m write chunk 32's
  // bytes 0..m-1 from lane 31's block (broadcast by shuffle)
  const bool head = lane < 16 - m, tail = lane >= 16 && lane < 16 + m;
  const unsigned src = tail ? 31u : 0u;
  const Block4 e{__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src),
                 __shfl_sync(0xffffffffu, v.z, src), __shfl_sync(0xffffffffu, v.w, src)};
  const unsigned b = head ? lane : (lane - 16) + (16 - m);  // byte index within the source block
  const std::uint32_t wv = b < 4 ? e.x : b < 8 ? e.y : b < 12 ? e.z : e.w;
  const std::uint8_t byte = static_cast<std::uint8_t>(wv >> (8 * (b & 3)));
  if (head) c[m + lane] = byte;
  else if (tail) c[512 + (lane - 16)] = byte;
}

// PKCS#7 always-pad block: tail bytes then k = 16 - tail_len copies of k.
__device__ __forceinline__ Block4 pad_block(const std::uint8_t* tail, std::uint32_t tail_len) {
  std::uint32_t w[4];
  const std::uint32_t k = 16u - tail_len;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    std::uint32_t v = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const std::uint32_t i = 4 * c + b;
      const std::uint32_t byte = i < tail_len ? tail[i] : k;
      v |= byte << (8 * b);
    }
    w[c] = v;
  }
  return Block4{w[0], w[1], w[2], w[3]};
}

// PKCS#7 trailer check of a decrypted last block (chunk.cpp:151-161).
__device__ __forceinline__ std::uint32_t pad_check(const Block4& b) {
  const std::uint32_t w[4] = {b.x, b.y, b.z, b.w};
  const std::uint32_t k = b.w >> 24;
  bool ok = k >= 1 && k <= 16;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const std::uint32_t byte = (w[i >> 2] >> (8 * (i & 3))) & 0xff;
    if (i >= 16 - static_cast<int>(k) && byte != k) ok = false;
  }
  return ok ? k : 0xffffffffu;
}

// ---------------------------------------------------------------- single key
template <bool DEC, int NB, bool ALIGNED>
__global__ void __launch_bounds__(kThreads, 1) ecb_kernel(const __grid_constant__ EcbArgs a) {
  extern __shared__ __align__(16) std::uint32_t sm[];
  const std::uint32_t lane = threadIdx.x & 31;
  const std::uint32_t lane4 = lane * 4;
  constexpr unsigned long long kTile = 32ull * NB;
  const unsigned long long ntiles = (a.nblocks + kTile - 1) / kTile;
  // tiles of whole input blocks; the tile holding the last block goes to the
  // ragged loop when the call checks a trailer or reports its result, so the
  // thread that owns that block always runs the epilogue
  const bool report = a.check_pad || a.result != nullptr;
  const unsigned long long full_tiles = ((report && a.nblocks == a.nfull) ? a.nfull - 1 : a.nfull) / kTile;
  const unsigned long long wpc = blockDim.x / 32;
  // tiles interleave across CTAs (tile t -> CTA t mod grid), so a short input
  // spreads over many SMs instead of queueing on one SM's lookup pipe
  unsigned long long tile = static_cast<unsigned long long>(threadIdx.x / 32) * gridDim.x + blockIdx.x;
  const unsigned long long tstride = gridDim.x * wpc;

  // steady state: whole tiles of whole input blocks, no per-block checks.
  // The next tile's blocks are loaded before the current tile is computed
  // (register double buffer), so a warp never waits on HBM at a tile start --
  // otherwise the SM's warps, which advance in near lockstep on short
  // launches, all stall on the same load latency together.  Without PDL the
  // first tile's loads are issued before the tables are staged, so their HBM
  // latency hides behind the staging; with PDL (the default) the staging
  // instead overlaps the previous launch's tail, and the loads wait for
  // griddepcontrol.wait.
  // Full tiles keep all 32 lanes active, so an output that is not even
  // 4-byte aligned is written by whole rows (store_row_unaligned).  Measured
  // on 1 GiB (scripts/unaligned_probe.py): per-lane double-chunk loads + word
  // stores at offsets 4/8 (753 GB/s) and + row stores at odd offsets (684)
  // beat cooperative shuffle loads (680 / 679) and byte stores (~400-570).
  const bool row_out = !ALIGNED && (reinterpret_cast<std::uintptr_t>(a.out) & 3) != 0;  // warp-uniform
  Block4 nxt[NB];
  auto load_tile = [&](unsigned long long t) {
#pragma unroll
    for (int j = 0; j < NB; ++j) nxt[j] = load_block<ALIGNED>(a.in + 16ull * (t * kTile + lane + 32ull * j));
  };
#if PAES_PDL
  // programmatic dependent launch: stage the tables (constant data) while the
  // previous kernel in the stream drains, let the next launch in, and touch
  // the buffers only once the previous grid has completed
#if PAES_PREFETCH
  // ...except for an L2 prefetch of the first tile: a hint with no
  // architectural effect (L2 is coherent for every SM and global stores write
  // through to it, so data the previous grid is still writing is read fresh
  // after the wait), it moves the tile's HBM latency under the staging
#pragma unroll
  for (int p = 0; p < PAES_PREFETCH; ++p) {
    const unsigned long long t = tile + p * tstride;
    if (t < full_tiles) {
#pragma unroll
      for (int j = 0; j < NB; ++j)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a.in + 16ull * (t * kTile + lane + 32ull * j)));
    }
  }
#endif
  stage_tables<DEC>(sm);
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (tile < full_tiles) load_tile(tile);
  __syncthreads();
#else
  if (tile < full_tiles) load_tile(tile);
  stage_tables<DEC>(sm);
  __syncthreads();
#endif
  const char* smb = reinterpret_cast<const char*>(sm);
  for (; tile < full_tiles; tile += tstride) {
    const unsigned long long b0 = tile * kTile + lane;
    Block4 s[NB];
#pragma unroll
    for (int j = 0; j < NB; ++j) s[j] = nxt[j];
    const unsigned long long next = tile + tstride;
    if (next < full_tiles) load_tile(next);
    cipher<DEC, NB>(s, a.k.w, smb, lane4);
    if (row_out) {
#pragma unroll
      for (int j = 0; j < NB; ++j) store_row_unaligned(a.out + 16ull * (b0 - lane + 32ull * j), s[j], lane);
    } else {
#pragma unroll
      for (int j = 0; j < NB; ++j) store_block<ALIGNED>(a.out + 16ull * (b0 + 32ull * j), s[j]);
    }
  }
  // the (at most one) ragged tile: partial blocks, pad block, trailer check
  for (; tile < ntiles; tile += tstride) {
    const unsigned long long b0 = tile * kTile + lane;
    Block4 s[NB];
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      const unsigned long long idx = b0 + 32ull * j;
      if (idx < a.nfull) s[j] = load_block<ALIGNED>(a.in + 16ull * idx);
      else if (idx < a.nblocks) s[j] = pad_block(a.in + 16ull * a.nfull, a.tail_len);
      else s[j] = Block4{0, 0, 0, 0};
    }
    cipher<DEC, NB>(s, a.k.w, smb, lane4);
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      const unsigned long long idx = b0 + 32ull * j;
      if (idx < a.nblocks) {
        store_block<ALIGNED>(a.out + 16ull * idx, s[j]);
        if (idx == a.nblocks - 1) {
          unsigned long long olen = 16ull * a.nblocks;
          if (DEC && a.check_pad) {
            const std::uint32_t k = pad_check(s[j]);
            if (a.status) *a.status = k;
            olen = k == 0xffffffffu ? ~0ull : olen - k;
          }
          if (a.result) *a.result = olen;
        }
      }
    }
  }
  if (a.done_flag) {  // uniform: the host spins on *done_flag (EcbArgs)
    // the CTA's writes, ordered before thread 0's system-scope fence by the
    // barrier (fences are cumulative: the cooperative-groups grid barrier
    // pattern), then the count; one fence per CTA, not one per thread
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      if (atomicAdd(a.done_ctr, 1u) == gridDim.x - 1) {
        *a.done_ctr = 0;  // ready for the next launch on the caller's stream (stream-ordered)
        __threadfence_system();
        *reinterpret_cast<volatile unsigned*>(a.done_flag) = a.done_seq;
      }
    }
  }
}

// ---------------------------------------------------------------- batch
// Persistent warps over a contiguous range of warp tiles.  Each message owns
// whole tiles (BatchMsg::first_tile), so a tile never mixes keys: a warp
// reloads its 44 key registers only when it moves to the next message, and
// the only per-block checks are on the message's ragged last tile.
template <bool DEC, int NB, bool ALIGNED>
__global__ void __launch_bounds__(kThreads, 1) batch_kernel(const __grid_constant__ BatchArgs a) {
  extern __shared__ __align__(16) std::uint32_t sm[];
  stage_tables<DEC>(sm);
  // programmatic dependent launch, as in ecb_kernel: the staging above
  // overlaps the previous kernel's tail; descriptors and data are touched
  // only after it has completed
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  __syncthreads();
  const char* smb = reinterpret_cast<const char*>(sm);
  const std::uint32_t lane = threadIdx.x & 31;
  const std::uint32_t lane4 = lane * 4;
  constexpr unsigned long long kTile = 32ull * NB;
  const unsigned long long nwarps = static_cast<unsigned long long>(gridDim.x) * (blockDim.x / 32);
  // warps numbered CTA-minor, so consecutive tile ranges land on different SMs
  const unsigned long long warp = static_cast<unsigned long long>(threadIdx.x / 32) * gridDim.x + blockIdx.x;
  const unsigned long long t_begin = a.total_tiles * warp / nwarps;
  const unsigned long long t_end = a.total_tiles * (warp + 1) / nwarps;
  if (t_begin >= t_end) return;

  // last message whose first tile is <= t_begin (binary search, warp-uniform)
  std::uint32_t m = 0;
  {
    std::uint32_t lo = 0, hi = a.nmsg;
    while (hi - lo > 1) {
      const std::uint32_t mid = (lo + hi) / 2;
      if (a.msgs[mid].first_tile <= t_begin) lo = mid;
      else hi = mid;
    }
    m = lo;
  }
  // The warp's range is walked message by message: a tight loop over the
  // message's whole tiles (pointer increments, one bound -- the same shape as
  // ecb_kernel's steady state), then its ragged last tile.  Keys and the
  // descriptor are loaded once per message and stay in registers.
  // (Per-tile descriptor arithmetic and branches cost ~50 extra warp
  // instructions per tile: batch_kernel ran 3.3 % behind ecb_kernel.)
  constexpr unsigned long long kTileBytes = 16ull * kTile;
  std::uint32_t kw[44];
  unsigned long long tile = t_begin;
  for (;;) {
    const BatchMsg msg = a.msgs[m];
    const unsigned long long msg_end = min(t_end, m + 1 < a.nmsg ? a.msgs[m + 1].first_tile : ~0ull);
    {
      const uint4* kp = reinterpret_cast<const uint4*>(a.keys + 44ull * m);
#pragma unroll
      for (int i = 0; i < 11; ++i) {
        const uint4 v = __ldg(kp + i);
        kw[4 * i] = v.x;
        kw[4 * i + 1] = v.y;
        kw[4 * i + 2] = v.z;
        kw[4 * i + 3] = v.w;
      }
    }
    // tiles of whole input blocks; the tile holding the message's last block
    // goes to the ragged loop when the trailer is checked or the length
    // reported, so the thread that owns that block runs the epilogue
    const unsigned long long excl = ((a.check_pad || a.out_lens) && msg.nblocks == msg.nfull) ? 1 : 0;
    const unsigned long long whole = msg.nfull >= excl ? (msg.nfull - excl) / kTile : 0;
    const unsigned long long full_end = min(msg_end, msg.first_tile + whole);
    const unsigned long long t0 = (tile - msg.first_tile) * kTile + lane;  // lane's first block in the message
    const std::uint8_t* src = a.in + msg.in_off + 16ull * t0;
    std::uint8_t* dst = a.out + msg.out_off + 16ull * t0;
    if (tile < full_end) {
      // register double buffer as in ecb_kernel: the next whole tile loads
      // while this one is computed (config 5, scripts/ab_batch.sh: encrypt
      // 834 -> 851 GB/s with this loop shape; decrypt +0.8 % from prefetching
      // too, which the old per-tile loop lost 0.5 % on)
      Block4 nxt[NB];
#pragma unroll
      for (int j = 0; j < NB; ++j) nxt[j] = load_block<ALIGNED>(src + 512ull * j);
      for (; tile < full_end; ++tile) {
        Block4 s[NB];
#pragma unroll
        for (int j = 0; j < NB; ++j) s[j] = nxt[j];
        if (tile + 1 < full_end) {
#pragma unroll
          for (int j = 0; j < NB; ++j) nxt[j] = load_block<ALIGNED>(src + kTileBytes + 512ull * j);
        }
        cipher<DEC, NB>(s, kw, smb, lane4);
#pragma unroll
        for (int j = 0; j < NB; ++j) store_block<ALIGNED>(dst + 512ull * j, s[j]);
        src += kTileBytes;
        dst += kTileBytes;
      }
    }
    // the message's last tile: partial blocks, pad block, trailer check
    for (; tile < msg_end; ++tile) {
      const unsigned long long tb = (tile - msg.first_tile) * kTile + lane;
      const std::uint8_t* msrc = a.in + msg.in_off;
      std::uint8_t* mdst = a.out + msg.out_off;
      Block4 s[NB];
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        const unsigned long long lb = tb + 32ull * j;
        if (lb < msg.nfull) s[j] = load_block<ALIGNED>(msrc + 16ull * lb);
        else if (lb < msg.nblocks) s[j] = pad_block(msrc + 16ull * msg.nfull, msg.tail_len);
        else s[j] = Block4{0, 0, 0, 0};
      }
      cipher<DEC, NB>(s, kw, smb, lane4);
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        const unsigned long long lb = tb + 32ull * j;
        if (lb < msg.nblocks) {
          store_block<ALIGNED>(mdst + 16ull * lb, s[j]);
          if (lb == msg.nblocks - 1) {
            unsigned long long olen = 16ull * msg.nblocks;
            if (DEC && a.check_pad) {
              const std::uint32_t k = pad_check(s[j]);
              if (a.status) a.status[m] = k;
              olen = k == 0xffffffffu ? ~0ull : olen - k;
            }
            if (a.out_lens) a.out_lens[m] = olen;
          }
        }
      }
    }
    if (tile >= t_end) break;
    // next message with tiles (messages own >= 1 tile each; skip defensively)
    do {
      ++m;
    } while (m + 1 < a.nmsg && a.msgs[m + 1].first_tile <= tile);
  }
}

// ---------------------------------------------------------------- single-state transforms
// The reference's public per-transform wrappers (aes.hpp:72-78,
// aes.cpp:194-227) over n independent states, one thread per state, byte-wise
// from the definitions: the KAT/test face of the cipher, not the bulk path.
// State byte i sits at row i % 4, column i / 4 (aes.hpp:24-36).
__device__ __forceinline__ std::uint32_t gf2(std::uint32_t a) { return ((a << 1) ^ ((a >> 7) * 0x1bu)) & 0xffu; }

__device__ __forceinline__ std::uint32_t gfmul(std::uint32_t a, std::uint32_t b) {
  std::uint32_t p = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    p ^= (b & 1u) ? a : 0u;
    a = gf2(a);
    b >>= 1;
  }
  return p;
}

__global__ void state_op_kernel(int op, std::uint8_t* states, unsigned long long n, StateKey rk) {
  const unsigned long long i = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  std::uint8_t* p = states + 16ull * i;
  std::uint32_t c[16], o[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) c[j] = p[j];
  // multipliers of one output row: {2,3,1,1} forward, {14,11,13,9} inverse
  const std::uint32_t m0 = op == PAES_OP_MIX_COLUMNS ? 2u : 14u, m1 = op == PAES_OP_MIX_COLUMNS ? 3u : 11u;
  const std::uint32_t m2 = op == PAES_OP_MIX_COLUMNS ? 1u : 13u, m3 = op == PAES_OP_MIX_COLUMNS ? 1u : 9u;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int row = j & 3, col = j >> 2;
    switch (op) {
      case PAES_OP_SUB_BYTES: o[j] = g_tab.sbox[c[j]]; break;
      case PAES_OP_INV_SUB_BYTES: o[j] = g_tab.inv_sbox[c[j]]; break;
      case PAES_OP_SHIFT_ROWS: o[j] = c[row + 4 * ((col + row) & 3)]; break;      // row r rotates left by r
      case PAES_OP_INV_SHIFT_ROWS: o[j] = c[row + 4 * ((col - row) & 3)]; break;  // ... and back right
      case PAES_OP_MIX_COLUMNS:
      case PAES_OP_INV_MIX_COLUMNS: {
        const int b = 4 * col;
        o[j] = gfmul(c[b + row], m0) ^ gfmul(c[b + ((row + 1) & 3)], m1) ^ gfmul(c[b + ((row + 2) & 3)], m2) ^
               gfmul(c[b + ((row + 3) & 3)], m3);
        break;
      }
      default: o[j] = c[j] ^ rk.b[j]; break;  // PAES_OP_ADD_ROUND_KEY
    }
  }
#pragma unroll
  for (int j = 0; j < 16; ++j) p[j] = static_cast<std::uint8_t>(o[j]);
}

// ---------------------------------------------------------------- utilities
__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// word i of the config-4 stream (oracle_counter_fill restates it on the CPU)
__device__ __forceinline__ unsigned long long counter_word(unsigned long long seed, unsigned long long i) {
  return mix64(seed * 0xD1B54A32D192ED03ull + (i + 1) * 0x9E3779B97F4A7C15ull);
}

__global__ void counter_fill_kernel(unsigned long long seed, unsigned long long word0, unsigned long long nwords,
                                    unsigned long long* out) {
  const unsigned long long stride = static_cast<unsigned long long>(gridDim.x) * blockDim.x;
  const unsigned long long npairs = nwords / 2;
  for (unsigned long long p = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x; p < npairs;
       p += stride) {
    const unsigned long long i = word0 + 2 * p;
    reinterpret_cast<ulonglong2*>(out)[p] = make_ulonglong2(counter_word(seed, i), counter_word(seed, i + 1));
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && (nwords & 1)) out[nwords - 1] = counter_word(seed, word0 + nwords - 1);
}

__global__ void checksum_kernel(const unsigned long long* buf, unsigned long long nwords, unsigned long long base,
                                unsigned long long* out) {
  const unsigned long long stride = static_cast<unsigned long long>(gridDim.x) * blockDim.x;
  unsigned long long acc = 0;
  for (unsigned long long i = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < nwords;
       i += stride)
    acc += mix64(buf[i] ^ ((base + i) * 0x9E3779B97F4A7C15ull));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, acc);
}

__global__ void mismatch_kernel(const uint4* a, const uint4* b, unsigned long long nblocks, unsigned long long* out) {
  const unsigned long long stride = static_cast<unsigned long long>(gridDim.x) * blockDim.x;
  unsigned int cnt = 0;
  for (unsigned long long i = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < nblocks;
       i += stride) {
    const uint4 x = a[i], y = b[i];
    cnt += (x.x != y.x) | (x.y != y.y) | (x.z != y.z) | (x.w != y.w);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(out, static_cast<unsigned long long>(cnt));
}

__global__ void put_u64_kernel(unsigned long long* p, unsigned long long v) { *p = v; }

template <class KernelT>
cudaError_t set_smem(KernelT k, int bytes) {
  return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

}  // namespace

// ---------------------------------------------------------------- launchers
#ifndef PAES_NB
#define PAES_NB 2
#endif
constexpr int kNB = PAES_NB;  // blocks per thread per warp tile

cudaError_t prepare_kernels() {
  cudaError_t e;
  if ((e = set_smem(ecb_kernel<false, kNB, true>, kEncLaunchSmem))) return e;
  if ((e = set_smem(ecb_kernel<false, kNB, false>, kEncLaunchSmem))) return e;
  if ((e = set_smem(ecb_kernel<true, kNB, true>, kDecLaunchSmem))) return e;
  if ((e = set_smem(ecb_kernel<true, kNB, false>, kDecLaunchSmem))) return e;
  if ((e = set_smem(batch_kernel<false, kNB, true>, kEncLaunchSmem))) return e;
  if ((e = set_smem(batch_kernel<true, kNB, true>, kDecLaunchSmem))) return e;
  if ((e = set_smem(batch_kernel<false, kNB, false>, kEncLaunchSmem))) return e;
  if ((e = set_smem(batch_kernel<true, kNB, false>, kDecLaunchSmem))) return e;
  return cudaSuccess;
}

// Every launch goes through cudaLaunchKernelEx, whose return value is the
// launch's own error: the calling thread's last-error state (which may hold a
// non-sticky error the caller has not consumed yet) is neither read nor
// cleared here.
template <class... KArgs, class... Args>
static cudaError_t launch_k(void (*k)(KArgs...), unsigned long long grid, int block, int smem, cudaStream_t stream,
                            bool pdl, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(static_cast<unsigned>(block));
  cfg.dynamicSmemBytes = static_cast<std::size_t>(smem);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  if (pdl) {
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  const cudaError_t e = cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
  if (e == cudaSuccess) g_launches.fetch_add(1, std::memory_order_relaxed);
  return e;
}

cudaError_t launch_ecb(bool dec, const EcbArgs& args, int sm_count, cudaStream_t stream) {
  if (args.nblocks == 0) return cudaSuccess;
  // one CTA per SM, or one per warp tile when there are fewer tiles than SMs
  const unsigned long long ntiles = (args.nblocks + 32ull * kNB - 1) / (32ull * kNB);
  const unsigned long long grid = ntiles < static_cast<unsigned long long>(sm_count) ? ntiles : sm_count;
  const bool aligned = ((reinterpret_cast<std::uintptr_t>(args.in) | reinterpret_cast<std::uintptr_t>(args.out)) & 15) == 0;
  const int smem = dec ? kDecLaunchSmem : kEncLaunchSmem;
  const bool pdl = PAES_PDL != 0;
  if (dec) return aligned ? launch_k(ecb_kernel<true, kNB, true>, grid, kThreads, smem, stream, pdl, args)
                          : launch_k(ecb_kernel<true, kNB, false>, grid, kThreads, smem, stream, pdl, args);
  return aligned ? launch_k(ecb_kernel<false, kNB, true>, grid, kThreads, smem, stream, pdl, args)
                 : launch_k(ecb_kernel<false, kNB, false>, grid, kThreads, smem, stream, pdl, args);
}

unsigned batch_tile_blocks() { return 32u * kNB; }

cudaError_t launch_batch(bool dec, const BatchArgs& args, int sm_count, cudaStream_t stream) {
  if (args.total_tiles == 0) return cudaSuccess;
  // one CTA per SM, or one per warp tile when there are fewer tiles than SMs
  const unsigned long long grid =
      args.total_tiles < static_cast<unsigned long long>(sm_count) ? args.total_tiles : sm_count;
  const int smem = dec ? kDecLaunchSmem : kEncLaunchSmem;
  const bool aligned =
      args.aligned && ((reinterpret_cast<std::uintptr_t>(args.in) | reinterpret_cast<std::uintptr_t>(args.out)) & 15) == 0;
  const bool pdl = PAES_PDL != 0;
  if (dec) return aligned ? launch_k(batch_kernel<true, kNB, true>, grid, kThreads, smem, stream, pdl, args)
                          : launch_k(batch_kernel<true, kNB, false>, grid, kThreads, smem, stream, pdl, args);
  return aligned ? launch_k(batch_kernel<false, kNB, true>, grid, kThreads, smem, stream, pdl, args)
                 : launch_k(batch_kernel<false, kNB, false>, grid, kThreads, smem, stream, pdl, args);
}

cudaError_t launch_state_op(int op, std::uint8_t* d_states, unsigned long long n, const StateKey& rk,
                            cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  return launch_k(state_op_kernel, (n + 255) / 256, 256, 0, stream, false, op, d_states, n, rk);
}

cudaError_t launch_counter_fill(unsigned long long seed, unsigned long long word0, unsigned long long nwords, void* out,
                                int sm_count, cudaStream_t stream) {
  if (nwords == 0) return cudaSuccess;
  return launch_k(counter_fill_kernel, sm_count * 4ull, 512, 0, stream, false, seed, word0, nwords,
                  static_cast<unsigned long long*>(out));
}

cudaError_t launch_checksum(const void* buf, unsigned long long nwords, unsigned long long base, unsigned long long* d_out,
                            int sm_count, cudaStream_t stream) {
  if (nwords == 0) return cudaSuccess;
  return launch_k(checksum_kernel, sm_count * 4ull, 512, 0, stream, false,
                  static_cast<const unsigned long long*>(buf), nwords, base, d_out);
}

cudaError_t launch_mismatch(const void* a, const void* b, unsigned long long nblocks, unsigned long long* d_out,
                            int sm_count, cudaStream_t stream) {
  if (nblocks == 0) return cudaSuccess;
  return launch_k(mismatch_kernel, sm_count * 4ull, 512, 0, stream, false, static_cast<const uint4*>(a),
                  static_cast<const uint4*>(b), nblocks, d_out);
}

cudaError_t launch_put_u64(unsigned long long* p, unsigned long long v, cudaStream_t stream) {
  return launch_k(put_u64_kernel, 1, 1, 0, stream, false, p, v);
}

unsigned long long launch_count() { return g_launches.load(std::memory_order_relaxed); }

}  // namespace paes_b200
