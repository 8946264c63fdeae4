// host_copy.cpp -- bulk host copies of the staged ring and the file writer.
//
// The staged ring moves every byte of a pageable call through host DRAM six
// times (caller buffer -> pinned slot -> DMA -> DMA -> pinned slot -> caller
// buffer); with ordinary stores each destination line is first read for
// ownership, two more DRAM passes.  Non-temporal (streaming) stores write
// whole lines without that read and keep the copy from evicting the source
// from the caches.  Large copies use them on CPUs with AVX2 (checked at run
// time); PAES_NT_COPY=0 selects plain memcpy (A/B).
#include "host_copy.hpp"

#include <immintrin.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>

namespace paes_b200 {

namespace {

__attribute__((target("avx2"))) void nt_copy_avx2(std::uint8_t* dst, const std::uint8_t* src, std::size_t n) {
  std::size_t head = (32 - reinterpret_cast<std::uintptr_t>(dst) % 32) % 32;
  if (head > n) head = n;
  std::memcpy(dst, src, head);
  dst += head, src += head, n -= head;
  const std::size_t body = n & ~std::size_t(127);
  for (std::size_t i = 0; i < body; i += 128) {
    const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i));
    const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 32));
    const __m256i c = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 64));
    const __m256i d = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 96));
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i), a);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 32), b);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 64), c);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 96), d);
  }
  _mm_sfence();  // streaming stores are weakly ordered: drain before anyone reads dst
  std::memcpy(dst + body, src + body, n - body);
}

bool use_nt() {
  static const bool on = [] {
    const char* e = std::getenv("PAES_NT_COPY");
    if (e && e[0] == '0') return false;
    __builtin_cpu_init();
    return __builtin_cpu_supports("avx2") != 0;
  }();
  return on;
}

}  // namespace

void bulk_copy(std::uint8_t* dst, const std::uint8_t* src, std::size_t n) {
  if (n >= kStreamCopyMin && use_nt()) nt_copy_avx2(dst, src, n);
  else std::memcpy(dst, src, n);
}

}  // namespace paes_b200
