// host_copy.hpp -- bulk host memcpy with streaming stores (host_copy.cpp).
#pragma once

#include <cstddef>
#include <cstdint>

namespace paes_b200 {

// Copies of at least this many bytes use non-temporal stores (when AVX2 is
// available and PAES_NT_COPY is not 0); shorter ones plain memcpy.
constexpr std::size_t kStreamCopyMin = 256u << 10;
void bulk_copy(std::uint8_t* dst, const std::uint8_t* src, std::size_t n);

}  // namespace paes_b200
