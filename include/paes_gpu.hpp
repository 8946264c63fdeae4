// paes_gpu.hpp -- C++20 face of libpaes_cuda.so with the reference library's
// signatures (header-only, over the C ABI in paes_cuda.h).
//
// A caller of the reference's proj/include/paes/{aes,chunk,exec,errors}.hpp
// swaps `paes::` for `paes::gpu::` (or adds ExecStrategy::Gpu to run_job, see
// INTEGRATION.md) and gets the same bytes back from the sm_100a kernels:
//
//   reference (proj/include/paes/...)            here
//   aes::Key128, aes::RoundKeySchedule          gpu::Key128, gpu::RoundKeySchedule   (aes.hpp:19-50)
//   aes::encrypt_ecb / decrypt_ecb              gpu::encrypt_ecb / decrypt_ecb       (aes.hpp:86-89)
//   aes::encrypt_block / decrypt_block          gpu::encrypt_block / decrypt_block   (aes.hpp:81-82)
//   aes::State, gf_xtime, gf_mul, sbox()        gpu::State, gf_xtime, gf_mul, sbox() (aes.hpp:24-70)
//   aes::sub_bytes ... add_round_key            gpu::sub_bytes ... add_round_key     (aes.hpp:72-78)
//   encrypt_chunk / decrypt_chunk               gpu::encrypt_chunk / decrypt_chunk   (exec.hpp:61-65)
//   plan_chunks / plan_decrypt_chunks           gpu::plan_chunks / ...               (chunk.hpp:37-47)
//   pad_final / unpad_final                     gpu::pad_final / unpad_final         (chunk.hpp:49-54)
//   run_job(JobSpec) + ExecStrategy             gpu::run_job (every strategy on GPU) (exec.hpp:18-51)
//   run_worker_chunk(WorkerChunkArgs)           gpu::run_worker_chunk                (exec.hpp:46-59)
//   assemble(plan, chunks)                      gpu::assemble                        (chunk.hpp:57-58)
//   Error / IoError / PaddingError / WorkerError  same names, same bases           (errors.hpp:8-33)
//
// Error codes from the C ABI are rethrown as the reference's exception types.
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <filesystem>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "paes_cuda.h"

namespace paes::gpu {

// ---- errors (errors.hpp:8-33) ---------------------------------------------
class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class IoError : public Error {
 public:
  explicit IoError(const std::string& what) : Error(what) {}
};
class PaddingError : public Error {
 public:
  using Error::Error;
};
class WorkerError : public Error {
 public:
  using Error::Error;
};

inline void check(long long rc) {
  if (rc >= 0) return;
  const std::string msg = paes_cuda_last_error();
  switch (rc) {
    case PAES_EINVAL: throw std::invalid_argument(msg);
    case PAES_EBADMSG: throw PaddingError(msg);
    case PAES_EIO: throw IoError(msg);
    case PAES_EWORKER: throw WorkerError(msg);
    default: throw Error(msg + " (paes_cuda code " + std::to_string(rc) + ")");
  }
}

// ---- keys (aes.hpp:13-50) ---------------------------------------------------
inline constexpr std::size_t kBlockSize = 16;
inline constexpr int kRounds = 10;
using Block = std::array<std::uint8_t, kBlockSize>;
using RoundKey = std::array<std::uint8_t, kBlockSize>;

struct Key128 {
  std::array<std::uint8_t, kBlockSize> bytes{};
  friend bool operator==(const Key128&, const Key128&) = default;
};

// Expanded on the host (north_star (1)); immutable, shareable across threads.
class RoundKeySchedule {
 public:
  explicit RoundKeySchedule(const Key128& key) { check(paes_cuda_expand_key(key.bytes.data(), rk_.data())); }
  RoundKey round_key(int round) const {
    RoundKey k{};
    for (std::size_t i = 0; i < kBlockSize; ++i) k[i] = rk_[16 * static_cast<std::size_t>(round) + i];
    return k;
  }
  static constexpr int size() { return kRounds + 1; }
  const std::uint8_t* data() const { return rk_.data(); }

 private:
  std::array<std::uint8_t, 176> rk_{};
};

inline RoundKeySchedule expand_key(const Key128& key) { return RoundKeySchedule(key); }

// ---- state and single-state transforms (aes.hpp:24-36, 52-78) ---------------
// Byte i of a block sits at row i%4, column i/4.
struct State {
  std::array<std::uint8_t, kBlockSize> cells{};  // cells[row + 4*col]

  static State from_block(const Block& b) { return State{b}; }
  Block to_block() const { return cells; }
  std::uint8_t& at(int row, int col) { return cells[static_cast<std::size_t>(row + 4 * col)]; }
  std::uint8_t at(int row, int col) const { return cells[static_cast<std::size_t>(row + 4 * col)]; }
  friend bool operator==(const State&, const State&) = default;
};

// GF(2^8) modulo x^8 + x^4 + x^3 + x + 1 (scalar helpers; the bulk path never calls them).
constexpr std::uint8_t gf_xtime(std::uint8_t a) {
  return static_cast<std::uint8_t>((a << 1) ^ ((a >> 7) ? 0x1b : 0x00));
}
constexpr std::uint8_t gf_mul(std::uint8_t a, std::uint8_t b) {
  std::uint8_t p = 0;
  for (; b; b >>= 1, a = gf_xtime(a))
    if (b & 1) p ^= a;
  return p;
}

namespace detail {
inline std::array<std::uint8_t, 256> table(int inverse) {
  std::array<std::uint8_t, 256> t{};
  check(paes_cuda_sbox(inverse, t.data()));
  return t;
}
inline State state_op(int op, State s, const std::uint8_t* rk = nullptr) {
  check(paes_cuda_state_transform(op, s.cells.data(), 1, rk));
  return s;
}
}  // namespace detail

inline const std::array<std::uint8_t, 256>& sbox() {
  static const auto t = detail::table(0);
  return t;
}
inline const std::array<std::uint8_t, 256>& inv_sbox() {
  static const auto t = detail::table(1);
  return t;
}

// Each runs on the GPU (paes_cuda_state_transform); batch many states with
// the C entry point directly.
inline State sub_bytes(State s) { return detail::state_op(PAES_OP_SUB_BYTES, s); }
inline State inv_sub_bytes(State s) { return detail::state_op(PAES_OP_INV_SUB_BYTES, s); }
inline State shift_rows(State s) { return detail::state_op(PAES_OP_SHIFT_ROWS, s); }
inline State inv_shift_rows(State s) { return detail::state_op(PAES_OP_INV_SHIFT_ROWS, s); }
inline State mix_columns(State s) { return detail::state_op(PAES_OP_MIX_COLUMNS, s); }
inline State inv_mix_columns(State s) { return detail::state_op(PAES_OP_INV_MIX_COLUMNS, s); }
inline State add_round_key(State s, const RoundKey& rk) {
  return detail::state_op(PAES_OP_ADD_ROUND_KEY, s, rk.data());
}

// ---- bulk ECB (aes.hpp:84-89): len % 16 == 0, in/out same length, may alias
inline void encrypt_ecb(std::span<const std::uint8_t> in, std::span<std::uint8_t> out, const RoundKeySchedule& ks,
                        int ngpus = 0) {
  if (in.size() != out.size() || in.size() % kBlockSize != 0)
    throw std::invalid_argument("encrypt_ecb: length must be a multiple of 16 and match output");
  check(paes_cuda_ecb(PAES_ENCRYPT, in.data(), out.data(), in.size(), ks.data(), ngpus));
}

inline void decrypt_ecb(std::span<const std::uint8_t> in, std::span<std::uint8_t> out, const RoundKeySchedule& ks,
                        int ngpus = 0) {
  if (in.size() != out.size() || in.size() % kBlockSize != 0)
    throw std::invalid_argument("decrypt_ecb: length must be a multiple of 16 and match output");
  check(paes_cuda_ecb(PAES_DECRYPT, in.data(), out.data(), in.size(), ks.data(), ngpus));
}

inline Block encrypt_block(const Block& in, const RoundKeySchedule& ks) {
  Block out{};
  encrypt_ecb(in, out, ks, 1);
  return out;
}

inline Block decrypt_block(const Block& in, const RoundKeySchedule& ks) {
  Block out{};
  decrypt_ecb(in, out, ks, 1);
  return out;
}

// ---- chunk transforms (exec.hpp:61-65) --------------------------------------
namespace detail {
// The result vector of a chunk transform.  `std::vector<uint8_t>(n)` zero-fills
// its n bytes on the calling thread before the engine overwrites every one of
// them: for a 4 GiB chunk that single-threaded fill (page faults included)
// costs several times the whole GPU call.  With libstdc++ the storage of a
// large result is therefore reserved and the size set without touching it, so
// its pages are first touched by the engine's parallel host copies (the same
// idea as folly::resizeWithoutInitialization; the reference's signature, a
// plain std::vector, is kept).  Other standard libraries, libstdc++'s debug
// and sanitizer-annotated vectors, small results and -DPAES_GPU_NO_UNINIT take
// the ordinary zero-filled vector.
inline std::vector<std::uint8_t> result_bytes(std::size_t n) {
#if defined(__GLIBCXX__) && !defined(_GLIBCXX_DEBUG) && !defined(_GLIBCXX_SANITIZE_VECTOR) && !defined(PAES_GPU_NO_UNINIT)
  if (n >= (std::size_t(1) << 20)) {
    struct Raw : std::vector<std::uint8_t> {
      void set_size_uninitialized(std::size_t m) {
        this->reserve(m);
        this->_M_impl._M_finish = this->_M_impl._M_start + m;
      }
    };
    Raw r;
    r.set_size_uninitialized(n);
    return std::vector<std::uint8_t>(std::move(r));
  }
#endif
  return std::vector<std::uint8_t>(n);
}
}  // namespace detail

inline std::vector<std::uint8_t> encrypt_chunk(std::span<const std::uint8_t> raw, bool is_final,
                                               const RoundKeySchedule& ks, int ngpus = 0) {
  if (!is_final && raw.size() % kBlockSize != 0)
    throw std::invalid_argument("non-final chunk length must be a multiple of 16");
  std::vector<std::uint8_t> out = detail::result_bytes(is_final ? (raw.size() / kBlockSize + 1) * kBlockSize : raw.size());
  std::uint64_t n = 0;
  check(paes_cuda_chunk(PAES_ENCRYPT, raw.data(), raw.size(), is_final ? 1 : 0, ks.data(), out.data(), &n, ngpus));
  out.resize(n);
  return out;
}

inline std::vector<std::uint8_t> decrypt_chunk(std::span<const std::uint8_t> cipher, bool is_final,
                                               const RoundKeySchedule& ks, int ngpus = 0) {
  std::vector<std::uint8_t> out = detail::result_bytes(cipher.size());
  std::uint64_t n = 0;
  check(paes_cuda_chunk(PAES_DECRYPT, cipher.data(), cipher.size(), is_final ? 1 : 0, ks.data(), out.data(), &n,
                        ngpus));
  out.resize(n);
  return out;
}

// ---- chunk planner (chunk.hpp:18-59) ----------------------------------------
inline constexpr std::uint64_t kBlock = 16;

struct ChunkSpec {
  std::uint64_t offset = 0, raw_len = 0, padded_len = 0;
  bool is_final = false;
  friend bool operator==(const ChunkSpec&, const ChunkSpec&) = default;
};

struct ChunkPlan {
  std::uint64_t total_len = 0;
  unsigned workers = 1;
  std::vector<ChunkSpec> chunks;
  std::uint64_t output_len() const {
    std::uint64_t s = 0;
    for (const auto& c : chunks) s += c.padded_len;
    return s;
  }
};

namespace detail {
template <class F>
ChunkPlan plan_with(F fn, std::uint64_t len, unsigned workers) {
  const std::int64_t n = fn(len, workers, nullptr, 0);
  check(n);
  std::vector<paes_chunk_spec> specs(static_cast<std::size_t>(n));
  check(fn(len, workers, specs.data(), specs.size()));
  ChunkPlan p{len, workers, {}};
  for (const auto& s : specs) p.chunks.push_back({s.offset, s.raw_len, s.padded_len, s.is_final != 0});
  return p;
}
}  // namespace detail

inline ChunkPlan plan_chunks(std::uint64_t total_len, unsigned workers) {
  return detail::plan_with(paes_cuda_plan_chunks, total_len, workers);
}
inline ChunkPlan plan_decrypt_chunks(std::uint64_t cipher_len, unsigned workers) {
  return detail::plan_with(paes_cuda_plan_decrypt_chunks, cipher_len, workers);
}

inline std::vector<std::uint8_t> pad_final(std::span<const std::uint8_t> raw) {
  std::vector<std::uint8_t> out((raw.size() / kBlock + 1) * kBlock);
  check(paes_cuda_pad_final(raw.data(), raw.size(), out.data()));
  return out;
}

inline std::size_t unpad_final(std::span<const std::uint8_t> padded) {
  const std::int64_t n = paes_cuda_unpad_final(padded.data(), padded.size());
  check(n);
  return static_cast<std::size_t>(n);
}

// Plain concatenation in plan order (chunk.cpp:102-111).
inline std::vector<std::uint8_t> assemble(const ChunkPlan& plan,
                                          const std::vector<std::vector<std::uint8_t>>& encrypted_chunks) {
  if (encrypted_chunks.size() != plan.chunks.size())
    throw std::invalid_argument("assemble: chunk count does not match plan");
  std::vector<std::uint8_t> out;
  out.reserve(static_cast<std::size_t>(plan.output_len()));
  for (const auto& c : encrypted_chunks) out.insert(out.end(), c.begin(), c.end());
  return out;
}

// ---- run_job with the GPU strategy (exec.hpp:18-51, exec.cpp:340-347) ------
enum class Direction { Encrypt, Decrypt };

// The reference's strategies plus the GPU one (exec.hpp:18, exec.cpp:24-38).
// Only Gpu runs here: the CPU strategies are the reference's own code.
enum class ExecStrategy { Sequential, Threaded, ProcessIsolated, Gpu };

constexpr std::string_view to_string(ExecStrategy s) {
  switch (s) {
    case ExecStrategy::Sequential: return "sequential";
    case ExecStrategy::Threaded: return "threads";
    case ExecStrategy::ProcessIsolated: return "processes";
    case ExecStrategy::Gpu: return "gpu";
  }
  return "gpu";
}

constexpr std::optional<ExecStrategy> strategy_from_string(std::string_view name) {
  if (name == "sequential") return ExecStrategy::Sequential;
  if (name == "threads") return ExecStrategy::Threaded;
  if (name == "processes") return ExecStrategy::ProcessIsolated;
  if (name == "gpu") return ExecStrategy::Gpu;
  return std::nullopt;
}

// Same members, order and defaults as the reference's JobSpec (exec.hpp:26-37),
// so aggregate and designated initialisers written for it compile unchanged;
// the Gpu strategy is opt-in, as a fourth ExecStrategy value would be.
struct JobSpec {
  std::filesystem::path input_path;
  std::filesystem::path output_path;
  Key128 key;
  unsigned workers = 1;  // Gpu strategy: GPUs, 0 = all visible
  ExecStrategy strategy = ExecStrategy::Sequential;
  Direction direction = Direction::Encrypt;
  std::filesystem::path worker_exe;  // unused by the GPU pipeline (kept for source compatibility)
};

struct JobOutcome {
  std::uint64_t bytes_in = 0;
  std::uint64_t bytes_out = 0;
  double seconds = 0.0;
};

// Every strategy runs the GPU file pipeline: the reference's CPU strategies
// write identical bytes (test_exec.cpp:64-86), so a JobSpec written for the
// reference keeps its strategy.  Their `workers` count CPU workers and are
// clamped to the visible GPUs; 0 keeps the reference's invalid_argument
// (exec.cpp:209, 273).  Sequential runs one shard and, like run_sequential
// (exec.cpp:206), raises a bad trailer as PaddingError, not WorkerError.
inline JobOutcome run_job(const JobSpec& job) {
  unsigned workers = job.workers;
  switch (job.strategy) {
    case ExecStrategy::Sequential: workers = 1; break;
    case ExecStrategy::Threaded:
    case ExecStrategy::ProcessIsolated: {
      if (workers == 0)
        throw std::invalid_argument(job.strategy == ExecStrategy::Threaded
                                        ? "run_threaded: workers must be >= 1"
                                        : "run_process_isolated: workers must be >= 1");
      const int n = paes_cuda_device_count();
      workers = std::max(1u, std::min(workers, static_cast<unsigned>(n > 0 ? n : 1)));
      break;
    }
    case ExecStrategy::Gpu: break;
  }
  paes_job_outcome o{};
  try {
    check(paes_cuda_run_job(job.input_path.c_str(), job.output_path.c_str(), job.key.bytes.data(), workers,
                            job.direction == Direction::Encrypt ? PAES_ENCRYPT : PAES_DECRYPT, &o));
  } catch (const WorkerError& e) {
    // "worker failure: chunk 0: unpad: ..." -> the inner PaddingError
    const std::string m = e.what();
    const auto p = m.find(": unpad:");
    if (job.strategy == ExecStrategy::Sequential && p != std::string::npos) throw PaddingError(m.substr(p + 2));
    throw;
  }
  return {o.bytes_in, o.bytes_out, o.seconds};
}

// One worker's chunk, file to file (exec.hpp:46-59, exec.cpp:349-373).
struct WorkerChunkArgs {
  std::filesystem::path input_path;
  std::uint64_t offset = 0;
  std::uint64_t raw_len = 0;
  bool is_final = false;
  Direction direction = Direction::Encrypt;
  Key128 key;
  std::filesystem::path out_path;
};

inline void run_worker_chunk(const WorkerChunkArgs& a, int device = -1) {
  check(paes_cuda_worker_chunk(a.input_path.c_str(), a.offset, a.raw_len, a.is_final ? 1 : 0,
                               a.direction == Direction::Encrypt ? PAES_ENCRYPT : PAES_DECRYPT, a.key.bytes.data(),
                               a.out_path.c_str(), device));
}

}  // namespace paes::gpu
