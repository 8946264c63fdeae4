// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" shim over the reference's own paes_core, compiled together with
// the reference sources where they lie (/root/reference/proj/src/*.cpp, never
// copied) by oracle/Makefile into oracle/_ref/libpaes_ref.so.  tests/ use it to
// pin the C restatement (oracle/aes_oracle.c) to the real reference, and
// bench.py uses it as the CPU baseline ("kind": "reference") and as the
// `--impl reference` arm.  Exceptions are mapped to negative codes exactly the
// way the product C-ABI maps them (include/paes_cuda.h).
#include <sys/stat.h>
#include <unistd.h>

#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <filesystem>
#include <fstream>
#include <span>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "paes/aes.hpp"
#include "paes/bench.hpp"
#include "paes/chunk.hpp"
#include "paes/errors.hpp"
#include "paes/exec.hpp"

namespace {

constexpr int kEINVAL = -22;
constexpr int kEBADMSG = -74;
constexpr int kEIO = -5;
constexpr int kEWORKER = -1001;
constexpr int kEOTHER = -1000;

paes::aes::Key128 to_key(const std::uint8_t* k) {
  paes::aes::Key128 key;
  std::memcpy(key.bytes.data(), k, 16);
  return key;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const paes::PaddingError&) {
    return kEBADMSG;
  } catch (const paes::WorkerError&) {
    return kEWORKER;
  } catch (const paes::IoError&) {
    return kEIO;
  } catch (const std::invalid_argument&) {
    return kEINVAL;
  } catch (...) {
    return kEOTHER;
  }
}

}  // namespace

extern "C" {

int ref_expand_key(const std::uint8_t* key, std::uint8_t* rk176) {
  return guarded([&] {
    const paes::aes::RoundKeySchedule ks(to_key(key));
    for (int r = 0; r < 11; ++r) std::memcpy(rk176 + 16 * r, ks.round_key(r).data(), 16);
  });
}

int ref_encrypt_block(const std::uint8_t* in, std::uint8_t* out, const std::uint8_t* key) {
  return guarded([&] {
    paes::aes::Block b;
    std::memcpy(b.data(), in, 16);
    const auto o = paes::aes::encrypt_block(b, paes::aes::RoundKeySchedule(to_key(key)));
    std::memcpy(out, o.data(), 16);
  });
}

int ref_decrypt_block(const std::uint8_t* in, std::uint8_t* out, const std::uint8_t* key) {
  return guarded([&] {
    paes::aes::Block b;
    std::memcpy(b.data(), in, 16);
    const auto o = paes::aes::decrypt_block(b, paes::aes::RoundKeySchedule(to_key(key)));
    std::memcpy(out, o.data(), 16);
  });
}

// aes::encrypt_ecb / decrypt_ecb (aes.hpp:86-89), single thread.
int ref_ecb(int dir, const std::uint8_t* in, std::uint8_t* out, std::uint64_t len, const std::uint8_t* key) {
  return guarded([&] {
    const paes::aes::RoundKeySchedule ks(to_key(key));
    std::span<const std::uint8_t> i(in, len);
    std::span<std::uint8_t> o(out, len);
    if (dir == 0) paes::aes::encrypt_ecb(i, o, ks);
    else paes::aes::decrypt_ecb(i, o, ks);
  });
}

// paes::encrypt_chunk / decrypt_chunk (exec.hpp:61-65).  `out` must hold len+16.
int ref_chunk(int dir, const std::uint8_t* in, std::uint64_t len, int is_final, const std::uint8_t* key,
              std::uint8_t* out, std::uint64_t* out_len) {
  return guarded([&] {
    const paes::aes::RoundKeySchedule ks(to_key(key));
    std::span<const std::uint8_t> i(in, len);
    const auto v = dir == 0 ? paes::encrypt_chunk(i, is_final != 0, ks) : paes::decrypt_chunk(i, is_final != 0, ks);
    if (!v.empty()) std::memcpy(out, v.data(), v.size());
    *out_len = v.size();
  });
}

// The reference's in-memory "pthreads" path (exec.cpp:143-202 without the
// file I/O): plan_chunks over `workers`, one std::thread per chunk, each
// running the reference's chunk transform into a disjoint output region.
int ref_threads(int dir, const std::uint8_t* in, std::uint64_t len, const std::uint8_t* key, std::uint8_t* out,
                std::uint64_t* out_len, unsigned workers) {
  return guarded([&] {
    const paes::aes::RoundKeySchedule ks(to_key(key));
    const auto plan = dir == 0 ? paes::plan_chunks(len, workers) : paes::plan_decrypt_chunks(len, workers);
    std::vector<std::string> failures(plan.chunks.size());
    std::vector<std::uint64_t> written(plan.chunks.size(), 0);
    std::vector<std::thread> pool;
    for (std::size_t idx = 0; idx < plan.chunks.size(); ++idx) {
      pool.emplace_back([&, idx] {
        try {
          const auto& c = plan.chunks[idx];
          std::span<const std::uint8_t> raw(in + c.offset, c.raw_len);
          std::span<std::uint8_t> dst(out + c.offset, c.padded_len);
          if (dir == 0) {
            if (c.is_final) {
              const auto v = paes::encrypt_chunk(raw, true, ks);  // pad_final + encrypt_ecb
              std::memcpy(dst.data(), v.data(), v.size());
            } else {
              paes::aes::encrypt_ecb(raw, dst, ks);
            }
            written[idx] = c.padded_len;
          } else {
            paes::aes::decrypt_ecb(raw, dst, ks);
            written[idx] = c.is_final ? paes::unpad_final(dst) : c.raw_len;
          }
        } catch (const std::exception& e) {
          failures[idx] = e.what();
        }
      });
    }
    for (auto& t : pool) t.join();
    std::string msg;
    for (std::size_t i = 0; i < failures.size(); ++i) {
      if (failures[i].empty()) continue;
      msg += (msg.empty() ? "" : "; ") + std::string("chunk ") + std::to_string(i) + ": " + failures[i];
    }
    if (!msg.empty()) throw paes::WorkerError("worker failure: " + msg);
    std::uint64_t tot = 0;
    for (auto w : written) tot += w;
    *out_len = tot;
  });
}

struct ref_chunk_spec {
  std::uint64_t offset, raw_len, padded_len;
  std::int32_t is_final, pad_;
};

long long ref_plan(int dir, std::uint64_t total_len, unsigned workers, ref_chunk_spec* out, std::uint64_t cap) {
  long long n = 0;
  const int rc = guarded([&] {
    const auto plan = dir == 0 ? paes::plan_chunks(total_len, workers) : paes::plan_decrypt_chunks(total_len, workers);
    if (plan.chunks.size() > cap) throw std::invalid_argument("cap");
    for (std::size_t i = 0; i < plan.chunks.size(); ++i) {
      const auto& c = plan.chunks[i];
      out[i] = ref_chunk_spec{c.offset, c.raw_len, c.padded_len, c.is_final ? 1 : 0, 0};
    }
    n = static_cast<long long>(plan.chunks.size());
  });
  return rc ? rc : n;
}

long long ref_unpad(const std::uint8_t* data, std::uint64_t len) {
  long long n = 0;
  const int rc = guarded([&] { n = static_cast<long long>(paes::unpad_final(std::span<const std::uint8_t>(data, len))); });
  return rc ? rc : n;
}

// bench.cpp:109-125 through a scratch file (the reference only writes files).
int ref_sweep(std::uint64_t seed, std::uint64_t size, std::uint8_t* out, const char* scratch_path) {
  return guarded([&] {
    paes::generate_sweep_file(scratch_path, size, seed);
    std::ifstream f(scratch_path, std::ios::binary);
    f.read(reinterpret_cast<char*>(out), static_cast<std::streamsize>(size));
    if (static_cast<std::uint64_t>(f.gcount()) != size) throw paes::IoError("short read", scratch_path);
    std::filesystem::remove(scratch_path);
  });
}

int ref_reject_outliers(const double* samples, std::uint64_t n, double* out, std::uint64_t* out_n) {
  return guarded([&] {
    const auto r = paes::reject_outliers(std::vector<double>(samples, samples + n));
    for (std::size_t i = 0; i < r.size(); ++i) out[i] = r[i];
    *out_n = r.size();
  });
}

unsigned ref_logical_cores() { return paes::logical_cores(); }
unsigned ref_physical_cores() { return paes::physical_cores(); }

// paes::run_job file->file (exec.cpp:340-347); strategy 0 seq, 1 threads.
int ref_run_job(const char* in_path, const char* out_path, const std::uint8_t* key, unsigned workers, int strategy,
                int dir, std::uint64_t* bytes_in, std::uint64_t* bytes_out, double* seconds) {
  return guarded([&] {
    paes::JobSpec job;
    job.input_path = in_path;
    job.output_path = out_path;
    job.key = to_key(key);
    job.workers = workers;
    job.strategy = strategy == 1 ? paes::ExecStrategy::Threaded : paes::ExecStrategy::Sequential;
    job.direction = dir == 0 ? paes::Direction::Encrypt : paes::Direction::Decrypt;
    const auto o = paes::run_job(job);
    *bytes_in = o.bytes_in;
    *bytes_out = o.bytes_out;
    *seconds = o.seconds;
  });
}

}  // extern "C"

extern "C" {

// run_job with any strategy (2 = ProcessIsolated, whose workers are spawned
// from `worker_exe`; exec.cpp:272-338) -- used to drive the GPU worker
// (paper_1403_7295_b200/lib/paes_gpu_worker) from the reference's own,
// unmodified process strategy.
int ref_run_job_ex(const char* in_path, const char* out_path, const std::uint8_t* key, unsigned workers, int strategy,
                   int dir, const char* worker_exe, std::uint64_t* bytes_in, std::uint64_t* bytes_out, double* seconds) {
  return guarded([&] {
    paes::JobSpec job;
    job.input_path = in_path;
    job.output_path = out_path;
    job.key = to_key(key);
    job.workers = workers;
    job.strategy = strategy == 2   ? paes::ExecStrategy::ProcessIsolated
                   : strategy == 1 ? paes::ExecStrategy::Threaded
                                   : paes::ExecStrategy::Sequential;
    job.direction = dir == 0 ? paes::Direction::Encrypt : paes::Direction::Decrypt;
    if (worker_exe && *worker_exe) job.worker_exe = worker_exe;
    const auto o = paes::run_job(job);
    *bytes_in = o.bytes_in;
    *bytes_out = o.bytes_out;
    *seconds = o.seconds;
  });
}

}  // extern "C"
