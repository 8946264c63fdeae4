// C++ tests of include/paes_gpu.hpp (the reference-signature shim over the
// C ABI), mirroring the reference's doctest cases.  Built and run by
// tests/test_cpp_shim.py:   test_shim host   (no GPU: planner, pad, keys, errors)
//                           test_shim gpu    (B200: ECB / chunk / run_job)
#include <unistd.h>

#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <random>
#include <string>
#include <vector>

#include "paes_gpu.hpp"

namespace gpu = paes::gpu;

static int g_fail = 0;
#define CHECK(c)                                                      \
  do {                                                                \
    if (!(c)) {                                                       \
      std::fprintf(stderr, "%s:%d CHECK failed: %s\n", __FILE__, __LINE__, #c); \
      ++g_fail;                                                       \
    }                                                                 \
  } while (0)

template <class E, class F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static std::vector<std::uint8_t> hex(const std::string& h) {
  std::vector<std::uint8_t> v;
  for (std::size_t i = 0; i + 1 < h.size(); i += 2) v.push_back(static_cast<std::uint8_t>(std::stoi(h.substr(i, 2), nullptr, 16)));
  return v;
}

static gpu::Key128 key_hex(const std::string& h) {
  gpu::Key128 k;
  const auto v = hex(h);
  std::copy(v.begin(), v.end(), k.bytes.begin());
  return k;
}

static void host_tests() {
  // key schedule KATs (test_aes.cpp:107-134)
  const gpu::RoundKeySchedule zero(gpu::Key128{});
  CHECK(zero.round_key(0) == gpu::RoundKey{});
  const auto r1 = zero.round_key(1);
  CHECK(std::vector<std::uint8_t>(r1.begin(), r1.end()) == hex("62636363626363636263636362636363"));
  const gpu::RoundKeySchedule fips(key_hex("2b7e151628aed2a6abf7158809cf4f3c"));
  CHECK(fips.round_key(1)[0] == 0xa0 && fips.round_key(1)[1] == 0xfa && fips.round_key(1)[2] == 0xfe &&
        fips.round_key(1)[3] == 0x17);
  // planner (test_chunk.cpp:57-117)
  auto p = gpu::plan_chunks(1000, 4);
  CHECK(p.chunks.size() == 4 && p.chunks[3].raw_len == 232 && p.chunks[3].padded_len == 240);
  CHECK(gpu::plan_chunks(16, 1).chunks[0].padded_len == 32);
  CHECK(gpu::plan_chunks(0, 33).chunks.size() == 1 && gpu::plan_chunks(0, 33).chunks[0].padded_len == 16);
  CHECK(gpu::plan_chunks(17, 33).chunks.size() == 2);
  CHECK(throws<std::invalid_argument>([] { gpu::plan_chunks(100, 0); }));
  for (std::uint64_t total : {0ull, 1ull, 15ull, 16ull, 17ull, 1000ull, 1024ull})
    for (unsigned w : {1u, 2u, 5u, 32u}) CHECK(gpu::plan_chunks(total, w).output_len() == (total / 16 + 1) * 16);
  auto d = gpu::plan_decrypt_chunks(1008, 4);
  CHECK(d.chunks.size() == 4 && d.chunks[0].raw_len == 256 && d.chunks[3].raw_len == 240 && d.chunks[3].is_final);
  CHECK(throws<gpu::PaddingError>([] { gpu::plan_decrypt_chunks(0, 2); }));
  CHECK(throws<gpu::PaddingError>([] { gpu::plan_decrypt_chunks(100, 2); }));
  CHECK(throws<std::invalid_argument>([] { gpu::plan_decrypt_chunks(1008, 0); }));
  // pad / unpad (test_chunk.cpp:128-163)
  CHECK(gpu::pad_final({}) == std::vector<std::uint8_t>(16, 0x10));
  std::vector<std::uint8_t> fifteen(15, 0xaa);
  CHECK(gpu::pad_final(fifteen).back() == 0x01);
  for (std::size_t len = 0; len <= 64; ++len) {
    std::vector<std::uint8_t> data(len);
    for (std::size_t i = 0; i < len; ++i) data[i] = static_cast<std::uint8_t>(i * 7 + 1);
    CHECK(gpu::unpad_final(gpu::pad_final(data)) == len);
  }
  CHECK(throws<gpu::PaddingError>([] { gpu::unpad_final({}); }));
  CHECK(throws<gpu::PaddingError>([] { gpu::unpad_final(std::vector<std::uint8_t>(16, 0x00)); }));
  CHECK(throws<gpu::PaddingError>([] { gpu::unpad_final(std::vector<std::uint8_t>(16, 0x11)); }));
  std::vector<std::uint8_t> inconsistent(16, 0x04);
  inconsistent[13] = 0x05;
  CHECK(throws<gpu::PaddingError>([&] { gpu::unpad_final(inconsistent); }));
  // GF(2^8) and the S-box tables (test_aes.cpp:55-105): FIPS-197 4.2 examples,
  // every S-box entry = affine(GF inverse), inverse table inverts it
  CHECK(gpu::gf_xtime(0x57) == 0xae && gpu::gf_mul(0x57, 0x83) == 0xc1 && gpu::gf_mul(0x57, 0x13) == 0xfe);
  const auto& sb = gpu::sbox();
  const auto& isb = gpu::inv_sbox();
  CHECK(sb[0x00] == 0x63 && sb[0x53] == 0xed);
  for (int x = 0; x < 256; ++x) {
    std::uint8_t inv = 0;
    for (int y = 1; y < 256 && x; ++y)
      if (gpu::gf_mul(static_cast<std::uint8_t>(x), static_cast<std::uint8_t>(y)) == 1) inv = static_cast<std::uint8_t>(y);
    std::uint8_t s = 0x63;
    for (int i = 0; i < 8; ++i) {
      const int bit = ((inv >> i) ^ (inv >> ((i + 4) % 8)) ^ (inv >> ((i + 5) % 8)) ^ (inv >> ((i + 6) % 8)) ^
                       (inv >> ((i + 7) % 8))) & 1;
      s ^= static_cast<std::uint8_t>(bit << i);
    }
    CHECK(sb[static_cast<std::size_t>(x)] == s);
    CHECK(isb[sb[static_cast<std::size_t>(x)]] == x);
  }
  // JobSpec: the reference's member order and defaults (exec.hpp:26-37), so its
  // designated initialisers compile and a default JobSpec is Sequential
  {
    const gpu::JobSpec d{.input_path = "/tmp/a", .output_path = "/tmp/b", .key = gpu::Key128{}, .workers = 3,
                         .strategy = gpu::ExecStrategy::Threaded, .direction = gpu::Direction::Decrypt,
                         .worker_exe = "/bin/true"};
    CHECK(d.workers == 3 && d.strategy == gpu::ExecStrategy::Threaded && d.direction == gpu::Direction::Decrypt);
    CHECK(gpu::JobSpec{}.strategy == gpu::ExecStrategy::Sequential && gpu::JobSpec{}.workers == 1);
  }
  // strategy names (exec.cpp:24-38) + "gpu"; the reference's worker-count rule (exec.cpp:209, 273)
  CHECK(gpu::to_string(gpu::ExecStrategy::Threaded) == "threads");
  CHECK(gpu::strategy_from_string("processes") == gpu::ExecStrategy::ProcessIsolated);
  CHECK(gpu::strategy_from_string("gpu") == gpu::ExecStrategy::Gpu);
  CHECK(!gpu::strategy_from_string("cuda").has_value());
  CHECK(throws<std::invalid_argument>([] {
    gpu::JobSpec j{"/tmp/a", "/tmp/b", gpu::Key128{}, 0, gpu::ExecStrategy::Threaded, gpu::Direction::Encrypt, {}};
    gpu::run_job(j);
  }));
  CHECK(throws<std::invalid_argument>([] {
    gpu::JobSpec j{"/tmp/a", "/tmp/b", gpu::Key128{}, 0, gpu::ExecStrategy::ProcessIsolated, gpu::Direction::Encrypt,
                   {}};
    gpu::run_job(j);
  }));
  // assemble (chunk.cpp:102-111): concatenation in plan order, count must match
  const auto plan3 = gpu::plan_chunks(100, 3);
  CHECK(gpu::assemble(plan3, {{1, 2}, {3}, {4, 5, 6}}) == std::vector<std::uint8_t>({1, 2, 3, 4, 5, 6}));
  CHECK(throws<std::invalid_argument>([&] { gpu::assemble(plan3, {{1}}); }));
  // run_worker_chunk: the input is checked first, IoError like exec.cpp:350-366
  CHECK(throws<gpu::IoError>([] {
    gpu::run_worker_chunk({"/nonexistent/paes_in", 0, 16, true, gpu::Direction::Encrypt, gpu::Key128{}, "/tmp/x"});
  }));
  // argument errors before any device work
  std::vector<std::uint8_t> fifteen_b(15), out(15);
  CHECK(throws<std::invalid_argument>([&] { gpu::encrypt_ecb(fifteen_b, out, zero); }));
  CHECK(throws<std::invalid_argument>([&] { gpu::encrypt_chunk(std::vector<std::uint8_t>(17), false, zero); }));
}

static void gpu_tests() {
  // FIPS-197 (test_aes.cpp:255-269)
  const gpu::RoundKeySchedule ks(key_hex("000102030405060708090a0b0c0d0e0f"));
  gpu::Block pt{};
  const auto pv = hex("00112233445566778899aabbccddeeff");
  std::copy(pv.begin(), pv.end(), pt.begin());
  const auto ct = gpu::encrypt_block(pt, ks);
  CHECK(std::vector<std::uint8_t>(ct.begin(), ct.end()) == hex("69c4e0d86a7b0430d8cdb78070b4c55a"));
  CHECK(gpu::decrypt_block(ct, ks) == pt);
  // zero-key snapshot (test_aes.cpp:285-292)
  const auto snap = gpu::decrypt_block(gpu::Block{}, gpu::RoundKeySchedule(gpu::Key128{}));
  CHECK(std::vector<std::uint8_t>(snap.begin(), snap.end()) == hex("140f0f1011b5223d79587717ffd9ec3a"));
  // ECB property (test_aes.cpp:294-312)
  std::vector<std::uint8_t> zeros(256, 0), enc(256), back(256);
  gpu::encrypt_ecb(zeros, enc, ks);
  const auto one = gpu::encrypt_block(gpu::Block{}, ks);
  for (int b = 0; b < 16; ++b) CHECK(std::equal(one.begin(), one.end(), enc.begin() + 16 * b));
  gpu::decrypt_ecb(enc, back, ks);
  CHECK(back == zeros);
  // chunk round trips across ragged sizes (test_exec.cpp:64-86, 139-155)
  std::mt19937_64 rng(101);
  // from 1 MiB up the result vectors are sized without being zero-filled first (detail::result_bytes)
  for (std::size_t n : {0ul, 1ul, 15ul, 16ul, 17ul, 31ul, 32ul, 1000ul, 65536ul, (1ul << 20) - 16, 1ul << 20, (1ul << 20) + 5,
                        (9ul << 20) + 3}) {
    std::vector<std::uint8_t> data(n);
    for (auto& x : data) x = static_cast<std::uint8_t>(rng());
    const auto c = gpu::encrypt_chunk(data, true, ks);
    CHECK(c.size() == (n / 16 + 1) * 16);
    CHECK(gpu::decrypt_chunk(c, true, ks) == data);
    if (n >= (1ul << 20)) {  // a failing call on the untouched-vector path: PaddingError, nothing leaked or torn
      gpu::Key128 other{};
      other.bytes[5] = 0x5a;
      CHECK(throws<gpu::PaddingError>([&] { gpu::decrypt_chunk(c, true, gpu::RoundKeySchedule(other)); }));
    }
    // region independence (test_exec.cpp:291-312): two chunks == one final chunk
    if (n >= 32 && n % 16 == 0) {
      const auto first = gpu::encrypt_chunk(std::span(data).subspan(0, 16), false, ks);
      const auto rest = gpu::encrypt_chunk(std::span(data).subspan(16), true, ks);
      CHECK(std::equal(first.begin(), first.end(), c.begin()));
      CHECK(std::equal(rest.begin(), rest.end(), c.begin() + 16));
    }
  }
  // single-state transforms on the GPU (test_aes.cpp:136-253)
  gpu::State st{};
  st.at(0, 0) = 0xdb, st.at(1, 0) = 0x13, st.at(2, 0) = 0x53, st.at(3, 0) = 0x45;
  const auto mc = gpu::mix_columns(st);
  CHECK(mc.at(0, 0) == 0x8e && mc.at(1, 0) == 0x4d && mc.at(2, 0) == 0xa1 && mc.at(3, 0) == 0xbc);
  gpu::State ones{};
  for (int r = 0; r < 4; ++r) ones.at(r, 2) = 0x01;
  CHECK(gpu::mix_columns(ones) == ones);
  gpu::State rows{};
  for (int r = 0; r < 4; ++r)
    for (int col = 0; col < 4; ++col) rows.at(r, col) = static_cast<std::uint8_t>(16 * r + col);
  const auto sr = gpu::shift_rows(rows);
  for (int r = 0; r < 4; ++r)
    for (int col = 0; col < 4; ++col) CHECK(sr.at(r, col) == rows.at(r, (col + r) % 4));
  std::mt19937_64 srng(147);
  for (int t = 0; t < 64; ++t) {
    gpu::State s{};
    gpu::RoundKey k{};
    for (auto& x : s.cells) x = static_cast<std::uint8_t>(srng());
    for (auto& x : k) x = static_cast<std::uint8_t>(srng());
    CHECK(gpu::inv_mix_columns(gpu::mix_columns(s)) == s);
    CHECK(gpu::inv_shift_rows(gpu::shift_rows(s)) == s);
    CHECK(gpu::inv_sub_bytes(gpu::sub_bytes(s)) == s);
    CHECK(gpu::add_round_key(gpu::add_round_key(s, k), k) == s);
    const auto sub = gpu::sub_bytes(s);
    for (std::size_t i = 0; i < 16; ++i) CHECK(sub.cells[i] == gpu::sbox()[s.cells[i]]);
  }
  // wrong key -> PaddingError (test_exec.cpp:235-247)
  std::vector<std::uint8_t> msg(100, 7);
  const auto c = gpu::encrypt_chunk(msg, true, ks);
  gpu::Key128 bad = key_hex("000102030405060708090a0b0c0d0e0f");
  bad.bytes[0] ^= 0xff;
  CHECK(throws<gpu::PaddingError>([&] { gpu::decrypt_chunk(c, true, gpu::RoundKeySchedule(bad)); }));
  // run_job (test_exec.cpp:139-155, 249-267) with the gpu strategy
  const auto dir = std::filesystem::temp_directory_path() / ("paes_shim_" + std::to_string(::getpid()));
  std::filesystem::create_directories(dir);
  std::vector<std::uint8_t> big(1 << 20);
  for (auto& x : big) x = static_cast<std::uint8_t>(rng());
  {
    std::ofstream f(dir / "mb.bin", std::ios::binary);
    f.write(reinterpret_cast<const char*>(big.data()), static_cast<std::streamsize>(big.size()));
  }
  gpu::JobSpec job{dir / "mb.bin", dir / "mb.enc", key_hex("000102030405060708090a0b0c0d0e0f"), 1,
                   gpu::ExecStrategy::Gpu, gpu::Direction::Encrypt};
  const auto o = gpu::run_job(job);
  CHECK(o.bytes_in == (1u << 20) && o.bytes_out == (1u << 20) + 16);
  gpu::JobSpec dec{dir / "mb.enc", dir / "mb.dec", job.key, 1, gpu::ExecStrategy::Gpu, gpu::Direction::Decrypt};
  CHECK(gpu::run_job(dec).bytes_out == (1u << 20));
  std::ifstream in(dir / "mb.dec", std::ios::binary);
  std::vector<std::uint8_t> got((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  CHECK(got == big);
  // run_worker_chunk over a 4-way plan, assembled == the whole-file ciphertext
  // (test_exec.cpp:291-312), then decrypted chunk by chunk
  const auto wplan = gpu::plan_chunks(big.size(), 4);
  std::vector<std::vector<std::uint8_t>> parts;
  for (std::size_t i = 0; i < wplan.chunks.size(); ++i) {
    const auto& c = wplan.chunks[i];
    const auto part = dir / ("part" + std::to_string(i));
    gpu::run_worker_chunk({dir / "mb.bin", c.offset, c.raw_len, c.is_final, gpu::Direction::Encrypt, job.key, part});
    std::ifstream pf(part, std::ios::binary);
    parts.emplace_back((std::istreambuf_iterator<char>(pf)), std::istreambuf_iterator<char>());
    CHECK(parts.back().size() == c.padded_len);
  }
  const auto whole = gpu::assemble(wplan, parts);
  CHECK(whole == gpu::encrypt_chunk(big, true, gpu::RoundKeySchedule(job.key)));
  const auto dplan = gpu::plan_decrypt_chunks(whole.size(), 3);
  std::vector<std::uint8_t> plain;
  for (std::size_t i = 0; i < dplan.chunks.size(); ++i) {
    const auto& c = dplan.chunks[i];
    const auto part = dir / ("plain" + std::to_string(i));
    gpu::run_worker_chunk({dir / "mb.enc", c.offset, c.raw_len, c.is_final, gpu::Direction::Decrypt, job.key, part});
    std::ifstream pf(part, std::ios::binary);
    plain.insert(plain.end(), std::istreambuf_iterator<char>(pf), std::istreambuf_iterator<char>());
  }
  CHECK(plain == big);
  gpu::Key128 wrong_key = job.key;
  wrong_key.bytes[3] ^= 0x40;
  const auto& last = dplan.chunks.back();
  CHECK(throws<gpu::PaddingError>([&] {
    gpu::run_worker_chunk(
        {dir / "mb.enc", last.offset, last.raw_len, true, gpu::Direction::Decrypt, wrong_key, dir / "bad.part"});
  }));
  CHECK(throws<gpu::IoError>([&] {  // chunk past the end of the file
    gpu::run_worker_chunk({dir / "mb.enc", whole.size() - 16, 32, true, gpu::Direction::Decrypt, job.key, dir / "x"});
  }));
  gpu::JobSpec wrong = dec;
  wrong.output_path = dir / "bad.dec";
  wrong.key.bytes[5] ^= 0x01;
  try {
    gpu::run_job(wrong);
    CHECK(false);
  } catch (const gpu::WorkerError& e) {
    CHECK(std::string(e.what()).find("chunk 0") != std::string::npos);
  }
  CHECK(!std::filesystem::exists(dir / "bad.dec"));
  // the reference's CPU strategy names run the same GPU pipeline, same bytes
  for (auto st : {gpu::ExecStrategy::Sequential, gpu::ExecStrategy::Threaded, gpu::ExecStrategy::ProcessIsolated}) {
    gpu::JobSpec j = job;
    j.output_path = dir / ("mb." + std::string(gpu::to_string(st)));
    j.workers = 4;
    j.strategy = st;
    CHECK(gpu::run_job(j).bytes_out == (1u << 20) + 16);
    std::ifstream f(j.output_path, std::ios::binary);
    CHECK(std::vector<std::uint8_t>((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>()) == whole);
  }
  wrong.strategy = gpu::ExecStrategy::Sequential;  // run_sequential: the PaddingError itself (exec.cpp:206)
  CHECK(throws<gpu::PaddingError>([&] { gpu::run_job(wrong); }));
  wrong.strategy = gpu::ExecStrategy::Threaded;
  CHECK(throws<gpu::WorkerError>([&] { gpu::run_job(wrong); }));
  CHECK(!std::filesystem::exists(dir / "bad.dec"));
  std::filesystem::remove_all(dir);
}

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "host";
  host_tests();
  if (mode == "gpu") gpu_tests();
  std::printf("%s: %s (%d failures)\n", mode.c_str(), g_fail ? "FAIL" : "ok", g_fail);
  return g_fail ? 1 : 0;
}
