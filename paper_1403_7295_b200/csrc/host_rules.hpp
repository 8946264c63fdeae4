// host_rules.hpp -- host-side C++ rules around the kernels: key expansion,
// the chunk planner (= the multi-GPU sharder), PKCS#7 pad/unpad, and the
// reference's seeded input generator.  Pure C++, no CUDA.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "aes_kernels.cuh"

namespace paes_b200 {

// Mirrors paes::PaddingError (errors.hpp:24-27).
struct PaddingError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Chunk {
  std::uint64_t offset = 0, raw_len = 0, padded_len = 0;
  bool is_final = false;
};

// RoundKeySchedule (aes.cpp:151-180): rk[16r + 4i + j] = w[4r+i][j].
void expand_key(const std::uint8_t key[16], std::uint8_t rk[176]);

// Kernel key words.  Encrypt: rk_0..rk_10 as little-endian column words.
// Decrypt (equivalent inverse cipher): rk_10, IMC(rk_9) .. IMC(rk_1), rk_0.
KeyWords enc_key_words(const std::uint8_t rk[176]);
KeyWords dec_key_words(const std::uint8_t rk[176]);

// plan_chunks / plan_decrypt_chunks (chunk.cpp:27-81).  Throw
// std::invalid_argument / PaddingError like the reference.
std::vector<Chunk> plan_chunks(std::uint64_t total_len, unsigned workers);
std::vector<Chunk> plan_decrypt_chunks(std::uint64_t cipher_len, unsigned workers);

// Shards a host-pointer call over `ndev` listed devices when the caller lets
// the library choose (ngpus = 0): at most one per kMinShardBytes of input,
// so a short call stays on one GPU instead of paying N launches and syncs.
constexpr std::uint64_t kMinShardBytes = 8ull << 20;
unsigned auto_shards(std::uint64_t len, unsigned ndev);

// unpad_final (chunk.cpp:90-100): unpadded length, throws PaddingError.
std::uint64_t unpad_final(const std::uint8_t* padded, std::uint64_t len);

// generate_sweep_file (bench.cpp:109-125) into memory.
void sweep(std::uint64_t seed, std::uint64_t size, std::uint8_t* out);

// Config-5 lengths.
void batch_lengths(std::uint64_t seed, std::uint32_t n, std::uint64_t* lens);

// Config-4 counter stream and the position-keyed checksum (host versions).
std::uint64_t counter_word(std::uint64_t seed, std::uint64_t i);
std::uint64_t checksum_words(const std::uint8_t* buf, std::uint64_t len, std::uint64_t base_word);

}  // namespace paes_b200
