// aes_tables.hpp -- compile-time AES-128 tables for the sm_100a kernels.
//
// The reference builds its S-box by brute-force GF(2^8) inversion plus the
// affine map (aes.cpp:10-39) and runs byte-wise rounds.  The GPU path uses the
// 32-bit T-table formulation instead: one table lookup per state byte per
// round gives SubBytes+ShiftRows+MixColumns at once.  Tables are generated here
// from log/antilog tables over the generator 0x03 (a different construction
// from the reference, so agreement with the oracle is a real check), and the
// word layout follows the reference's State contract (aes.hpp:24-36): byte i
// of a block is row i%4 of column i/4, so a little-endian uint32 load of bytes
// 4c..4c+3 is column c with row 0 in the low byte.
//
//   Te0[x] = {02.S[x], S[x], S[x], 03.S[x]}      (row 0 .. row 3, LE word)
//   Td0[x] = {0e.Si[x], 09.Si[x], 0d.Si[x], 0b.Si[x]}
//   Te_k = rotl(Te0, 8k), Td_k = rotl(Td0, 8k)  (built when staging into smem)
#pragma once

#include <cstdint>

namespace paes_b200 {

struct AesTables {
  std::uint8_t sbox[256];
  std::uint8_t inv_sbox[256];
  std::uint32_t te0[256];
  std::uint32_t td0[256];
};

namespace detail {

constexpr std::uint8_t xt(std::uint8_t a) { return static_cast<std::uint8_t>((a << 1) ^ ((a >> 7) * 0x1b)); }

constexpr std::uint8_t mul(std::uint8_t a, std::uint8_t b) {
  std::uint8_t p = 0;
  while (b) {
    if (b & 1) p ^= a;
    a = xt(a);
    b >>= 1;
  }
  return p;
}

constexpr AesTables make_tables() {
  AesTables t{};
  // antilog/log over generator 3
  std::uint8_t alog[256]{}, log[256]{};
  std::uint8_t v = 1;
  for (int i = 0; i < 255; ++i) {
    alog[i] = v;
    log[v] = static_cast<std::uint8_t>(i);
    v = static_cast<std::uint8_t>(v ^ xt(v));  // v *= 3
  }
  for (int x = 0; x < 256; ++x) {
    const std::uint8_t inv = x == 0 ? 0 : alog[(255 - log[x]) % 255];
    // affine map b ^ rotl1 ^ rotl2 ^ rotl3 ^ rotl4 ^ 0x63
    std::uint32_t r = inv;
    r ^= (r << 1) ^ (r << 2) ^ (r << 3) ^ (r << 4);
    const std::uint8_t s = static_cast<std::uint8_t>((r ^ (r >> 8) ^ 0x63) & 0xff);
    t.sbox[x] = s;
    t.inv_sbox[s] = static_cast<std::uint8_t>(x);
  }
  for (int x = 0; x < 256; ++x) {
    const std::uint8_t s = t.sbox[x], si = t.inv_sbox[x];
    t.te0[x] = static_cast<std::uint32_t>(mul(s, 2)) | (static_cast<std::uint32_t>(s) << 8) |
               (static_cast<std::uint32_t>(s) << 16) | (static_cast<std::uint32_t>(mul(s, 3)) << 24);
    t.td0[x] = static_cast<std::uint32_t>(mul(si, 0x0e)) | (static_cast<std::uint32_t>(mul(si, 0x09)) << 8) |
               (static_cast<std::uint32_t>(mul(si, 0x0d)) << 16) | (static_cast<std::uint32_t>(mul(si, 0x0b)) << 24);
  }
  return t;
}

}  // namespace detail

inline constexpr AesTables kTables = detail::make_tables();

static_assert(kTables.sbox[0x00] == 0x63 && kTables.sbox[0x53] == 0xed, "S-box spot entries (aes.cpp:53)");
static_assert(kTables.inv_sbox[0x63] == 0x00 && kTables.inv_sbox[0xed] == 0x53, "inverse S-box");
static_assert(kTables.te0[0x00] == 0xa56363c6u, "Te0[0] = {c6,63,63,a5}");
static_assert(kTables.td0[0x00] == 0x50a7f451u, "Td0[0] = {51,f4,a7,50}");

// GF(2^8) multiples {09,0b,0d,0e} x x for the host-side key transform.
struct InvMixTables {
  std::uint8_t m9[256], mb[256], md[256], me[256];
};

constexpr InvMixTables make_inv_mix_tables() {
  InvMixTables t{};
  for (int x = 0; x < 256; ++x) {
    const auto b = static_cast<std::uint8_t>(x);
    t.m9[x] = detail::mul(b, 0x09);
    t.mb[x] = detail::mul(b, 0x0b);
    t.md[x] = detail::mul(b, 0x0d);
    t.me[x] = detail::mul(b, 0x0e);
  }
  return t;
}

inline constexpr InvMixTables kInvMix = make_inv_mix_tables();

// InvMixColumns of one column word (used to derive the equivalent inverse
// cipher's round keys dk_r = InvMixColumns(rk_r), r = 1..9).  Table-driven:
// the batch path transforms 36 words per message for thousands of messages.
inline std::uint32_t inv_mix_column_word(std::uint32_t w) {
  const std::uint8_t a0 = w & 0xff, a1 = (w >> 8) & 0xff, a2 = (w >> 16) & 0xff, a3 = w >> 24;
  const InvMixTables& t = kInvMix;
  const std::uint32_t r0 = t.me[a0] ^ t.mb[a1] ^ t.md[a2] ^ t.m9[a3];
  const std::uint32_t r1 = t.m9[a0] ^ t.me[a1] ^ t.mb[a2] ^ t.md[a3];
  const std::uint32_t r2 = t.md[a0] ^ t.m9[a1] ^ t.me[a2] ^ t.mb[a3];
  const std::uint32_t r3 = t.mb[a0] ^ t.md[a1] ^ t.m9[a2] ^ t.me[a3];
  return r0 | (r1 << 8) | (r2 << 16) | (r3 << 24);
}

// Reference formulation kept for the compile-time self-check below.
constexpr std::uint32_t inv_mix_column_word_slow(std::uint32_t w) {
  const std::uint8_t a0 = w & 0xff, a1 = (w >> 8) & 0xff, a2 = (w >> 16) & 0xff, a3 = w >> 24;
  using detail::mul;
  const std::uint8_t r0 = mul(a0, 0x0e) ^ mul(a1, 0x0b) ^ mul(a2, 0x0d) ^ mul(a3, 0x09);
  const std::uint8_t r1 = mul(a0, 0x09) ^ mul(a1, 0x0e) ^ mul(a2, 0x0b) ^ mul(a3, 0x0d);
  const std::uint8_t r2 = mul(a0, 0x0d) ^ mul(a1, 0x09) ^ mul(a2, 0x0e) ^ mul(a3, 0x0b);
  const std::uint8_t r3 = mul(a0, 0x0b) ^ mul(a1, 0x0d) ^ mul(a2, 0x09) ^ mul(a3, 0x0e);
  return static_cast<std::uint32_t>(r0) | (static_cast<std::uint32_t>(r1) << 8) | (static_cast<std::uint32_t>(r2) << 16) |
         (static_cast<std::uint32_t>(r3) << 24);
}

static_assert(inv_mix_column_word_slow(0x01010101u) == 0x01010101u, "InvMixColumns fixes the all-ones column");
static_assert(kInvMix.me[0x01] == 0x0e && kInvMix.m9[0x80] == detail::mul(0x80, 0x09) && kInvMix.md[0xff] == detail::mul(0xff, 0x0d),
              "InvMixColumns multiply tables");

}  // namespace paes_b200
