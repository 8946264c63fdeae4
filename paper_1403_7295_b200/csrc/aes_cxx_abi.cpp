// aes_cxx_abi.cpp -- libpaes_aes_b200.so: the reference's aes.cpp entry points
// (include/paes/aes.hpp:39-89) as exported C++ symbols with the reference's
// exact mangled names and calling convention, each backed by libpaes_cuda.so.
//
// A program built from the reference's OTHER sources (chunk.cpp, exec.cpp,
// bench.cpp, report.cpp, python/paes_module.cpp -- unmodified) links against
// this library instead of compiling aes.cpp, and its whole chunked file path
// (encrypt_chunk_into -> aes::encrypt_ecb, exec.cpp:111-127; run_job's
// sequential / threaded / process strategies, exec.cpp:143-338) then runs the
// B200 kernels: a link-level drop-in with no source change on the reference
// side (oracle/Makefile target `linked`, tests/test_reference_smoke.py).
//
// The declarations below restate aes.hpp's interface because the ABI must
// match it: the same namespace, class names, member layout (RoundKeySchedule
// = 11 x 16 contiguous bytes, round r at byte 16r, FIPS order -- the 176-byte
// layout paes_cuda_expand_key writes) and parameter types (std::span by
// value, State by value).  Key expansion stays on the host (north_star (1));
// bulk ECB goes through paes_cuda_ecb (sharded over the listed GPUs, pageable
// spans staged by the library's pinned ring); the single-state transforms run
// the GPU state-op kernel.  Errors: std::invalid_argument with the reference's
// messages for shape errors (aes.cpp:243-245, 256-258), std::runtime_error for
// a device failure -- never a silent CPU path.
#include <array>
#include <cstddef>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>

#include "paes_cuda.h"

namespace paes::aes {

inline constexpr std::size_t kBlockSize = 16;
inline constexpr int kRounds = 10;
using Block = std::array<std::uint8_t, kBlockSize>;
using RoundKey = std::array<std::uint8_t, kBlockSize>;

struct Key128 {
  std::array<std::uint8_t, kBlockSize> bytes{};
};

struct State {
  std::array<std::uint8_t, kBlockSize> cells{};
};

class RoundKeySchedule {
 public:
  explicit RoundKeySchedule(const Key128& key);
  const std::uint8_t* data() const { return keys_[0].data(); }

 private:
  std::array<RoundKey, kRounds + 1> keys_{};
};

static_assert(sizeof(RoundKeySchedule) == 176 && sizeof(State) == 16 && sizeof(Key128) == 16,
              "layouts must match aes.hpp");

namespace {

void check(int rc) {
  if (rc == PAES_OK) return;
  const std::string msg = paes_cuda_last_error();
  if (rc == PAES_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error("paes_cuda: " + msg + " (code " + std::to_string(rc) + ")");
}

State state_op(int op, State s, const std::uint8_t* rk16 = nullptr) {
  check(paes_cuda_state_transform(op, s.cells.data(), 1, rk16));
  return s;
}

std::array<std::uint8_t, 256> table(int inverse) {
  std::array<std::uint8_t, 256> t{};
  check(paes_cuda_sbox(inverse, t.data()));
  return t;
}

// One GPU for a 16-byte block (no sharding decision to make).
Block block_op(int dir, const Block& in, const RoundKeySchedule& ks) {
  Block out{};
  check(paes_cuda_ecb(dir, in.data(), out.data(), kBlockSize, ks.data(), 1));
  return out;
}

void ecb(int dir, std::span<const std::uint8_t> in, std::span<std::uint8_t> out, const RoundKeySchedule& ks,
         const char* what) {
  if (in.size() != out.size() || in.size() % kBlockSize != 0)
    throw std::invalid_argument(std::string(what) + ": length must be a multiple of 16 and match output");
  if (in.empty()) return;
  // ngpus = 0: every listed GPU, at most one per 8 MiB (paes_cuda_auto_shards)
  check(paes_cuda_ecb(dir, in.data(), out.data(), in.size(), ks.data(), 0));
}

}  // namespace

RoundKeySchedule::RoundKeySchedule(const Key128& key) { check(paes_cuda_expand_key(key.bytes.data(), keys_[0].data())); }

RoundKeySchedule expand_key(const Key128& key) { return RoundKeySchedule(key); }

const std::array<std::uint8_t, 256>& sbox() {
  static const auto t = table(0);
  return t;
}

const std::array<std::uint8_t, 256>& inv_sbox() {
  static const auto t = table(1);
  return t;
}

State sub_bytes(State s) { return state_op(PAES_OP_SUB_BYTES, s); }
State inv_sub_bytes(State s) { return state_op(PAES_OP_INV_SUB_BYTES, s); }
State shift_rows(State s) { return state_op(PAES_OP_SHIFT_ROWS, s); }
State inv_shift_rows(State s) { return state_op(PAES_OP_INV_SHIFT_ROWS, s); }
State mix_columns(State s) { return state_op(PAES_OP_MIX_COLUMNS, s); }
State inv_mix_columns(State s) { return state_op(PAES_OP_INV_MIX_COLUMNS, s); }
State add_round_key(State s, const RoundKey& rk) { return state_op(PAES_OP_ADD_ROUND_KEY, s, rk.data()); }

Block encrypt_block(const Block& in, const RoundKeySchedule& ks) { return block_op(PAES_ENCRYPT, in, ks); }
Block decrypt_block(const Block& in, const RoundKeySchedule& ks) { return block_op(PAES_DECRYPT, in, ks); }

void encrypt_ecb(std::span<const std::uint8_t> in, std::span<std::uint8_t> out, const RoundKeySchedule& ks) {
  ecb(PAES_ENCRYPT, in, out, ks, "encrypt_ecb");
}

void decrypt_ecb(std::span<const std::uint8_t> in, std::span<std::uint8_t> out, const RoundKeySchedule& ks) {
  ecb(PAES_DECRYPT, in, out, ks, "decrypt_ecb");
}

}  // namespace paes::aes
