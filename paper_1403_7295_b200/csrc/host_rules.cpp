// host_rules.cpp -- see host_rules.hpp.
#include "host_rules.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <random>

#include "aes_tables.hpp"

namespace paes_b200 {

void expand_key(const std::uint8_t key[16], std::uint8_t rk[176]) {
  // Word-oriented FIPS-197 5.2 expansion; RotWord+SubWord+Rcon every 4th word.
  std::uint8_t w[44][4];
  std::memcpy(w, key, 16);
  std::uint8_t rcon = 1;
  for (int i = 4; i < 44; ++i) {
    std::uint8_t t[4] = {w[i - 1][0], w[i - 1][1], w[i - 1][2], w[i - 1][3]};
    if ((i & 3) == 0) {
      const std::uint8_t t0 = t[0];
      t[0] = static_cast<std::uint8_t>(kTables.sbox[t[1]] ^ rcon);
      t[1] = kTables.sbox[t[2]];
      t[2] = kTables.sbox[t[3]];
      t[3] = kTables.sbox[t0];
      rcon = static_cast<std::uint8_t>((rcon << 1) ^ ((rcon >> 7) * 0x1b));
    }
    for (int j = 0; j < 4; ++j) w[i][j] = static_cast<std::uint8_t>(w[i - 4][j] ^ t[j]);
  }
  std::memcpy(rk, w, 176);  // w is row-major [44][4] == keys_[r][4i+j] layout
}

static std::uint32_t le32(const std::uint8_t* p) {
  return static_cast<std::uint32_t>(p[0]) | (static_cast<std::uint32_t>(p[1]) << 8) |
         (static_cast<std::uint32_t>(p[2]) << 16) | (static_cast<std::uint32_t>(p[3]) << 24);
}

KeyWords enc_key_words(const std::uint8_t rk[176]) {
  KeyWords k{};
  for (int i = 0; i < 44; ++i) k.w[i] = le32(rk + 4 * i);
  return k;
}

KeyWords dec_key_words(const std::uint8_t rk[176]) {
  KeyWords k{};
  for (int c = 0; c < 4; ++c) k.w[c] = le32(rk + 160 + 4 * c);
  for (int i = 1; i <= 9; ++i) {
    const int r = 10 - i;
    for (int c = 0; c < 4; ++c) k.w[4 * i + c] = inv_mix_column_word(le32(rk + 16 * r + 4 * c));
  }
  for (int c = 0; c < 4; ++c) k.w[40 + c] = le32(rk + 4 * c);
  return k;
}

static std::vector<std::uint64_t> shares(std::uint64_t blocks, std::uint64_t n) {
  std::vector<std::uint64_t> s(n, blocks / n);
  for (std::uint64_t i = 0; i < blocks % n; ++i) s[i] += 1;  // larger shares first
  return s;
}

std::vector<Chunk> plan_chunks(std::uint64_t total_len, unsigned workers) {
  if (workers == 0) throw std::invalid_argument("plan_chunks: workers must be >= 1");
  const std::uint64_t data_blocks = (total_len + 15) / 16;
  const std::uint64_t n = std::min<std::uint64_t>(workers, std::max<std::uint64_t>(1, data_blocks));
  const auto sh = shares(data_blocks, n);
  std::vector<Chunk> plan(n);
  std::uint64_t off = 0;
  for (std::uint64_t i = 0; i < n; ++i) {
    Chunk& c = plan[i];
    c.offset = off;
    c.is_final = i + 1 == n;
    c.raw_len = c.is_final ? total_len - off : sh[i] * 16;
    c.padded_len = c.is_final ? (c.raw_len / 16 + 1) * 16 : c.raw_len;
    off += c.raw_len;
  }
  return plan;
}

std::vector<Chunk> plan_decrypt_chunks(std::uint64_t cipher_len, unsigned workers) {
  if (workers == 0) throw std::invalid_argument("plan_decrypt_chunks: workers must be >= 1");
  if (cipher_len == 0 || cipher_len % 16 != 0)
    throw PaddingError("ciphertext length must be a non-zero multiple of 16");
  const std::uint64_t blocks = cipher_len / 16;
  const std::uint64_t n = std::min<std::uint64_t>(workers, blocks);
  const auto sh = shares(blocks, n);
  std::vector<Chunk> plan(n);
  std::uint64_t off = 0;
  for (std::uint64_t i = 0; i < n; ++i) {
    Chunk& c = plan[i];
    c.offset = off;
    c.raw_len = c.padded_len = sh[i] * 16;
    c.is_final = i + 1 == n;
    off += c.raw_len;
  }
  return plan;
}

unsigned auto_shards(std::uint64_t len, unsigned ndev) {
  const std::uint64_t by_size = std::max<std::uint64_t>(1, len / kMinShardBytes);
  return static_cast<unsigned>(std::min<std::uint64_t>(std::max(1u, ndev), by_size));
}

std::uint64_t unpad_final(const std::uint8_t* padded, std::uint64_t len) {
  if (len == 0 || len % 16 != 0) throw PaddingError("unpad: length must be a non-zero multiple of 16");
  const std::uint8_t k = padded[len - 1];
  if (k == 0 || k > 16) throw PaddingError("unpad: invalid pad byte");
  for (std::uint64_t i = len - k; i < len; ++i)
    if (padded[i] != k) throw PaddingError("unpad: inconsistent pad bytes");
  return len - k;
}

void sweep(std::uint64_t seed, std::uint64_t size, std::uint8_t* out) {
  std::seed_seq seq{seed, size};  // same construction as bench.cpp:110-111
  std::mt19937_64 rng(seq);
  std::uint64_t off = 0;
  while (off < size) {
    const std::uint64_t w = rng();
    const std::uint64_t n = std::min<std::uint64_t>(8, size - off);
    for (std::uint64_t b = 0; b < n; ++b) out[off + b] = static_cast<std::uint8_t>(w >> (8 * b));
    off += n;
  }
}

void batch_lengths(std::uint64_t seed, std::uint32_t n, std::uint64_t* lens) {
  std::seed_seq seq{seed};
  std::mt19937_64 rng(seq);
  for (std::uint32_t i = 0; i < n; ++i) {
    const double u = static_cast<double>(rng() >> 11) * (1.0 / 9007199254740992.0);
    const double L = 4096.0 * std::exp2(10.0 * u);
    std::uint64_t r = static_cast<std::uint64_t>(std::floor(L / 16.0 + 0.5)) * 16;
    lens[i] = std::clamp<std::uint64_t>(r, 4096, 4194304);
  }
}

static std::uint64_t mix64(std::uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

std::uint64_t counter_word(std::uint64_t seed, std::uint64_t i) {
  return mix64(seed * 0xD1B54A32D192ED03ull + (i + 1) * 0x9E3779B97F4A7C15ull);
}

std::uint64_t checksum_words(const std::uint8_t* buf, std::uint64_t len, std::uint64_t base_word) {
  std::uint64_t acc = 0;
  for (std::uint64_t i = 0; i < len / 8; ++i) {
    std::uint64_t w;
    std::memcpy(&w, buf + 8 * i, 8);
    acc += mix64(w ^ ((base_word + i) * 0x9E3779B97F4A7C15ull));
  }
  return acc;
}

}  // namespace paes_b200
