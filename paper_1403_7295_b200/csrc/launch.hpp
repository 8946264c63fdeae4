// launch.hpp -- host-side launchers for the kernels in aes_kernels.cu.
#pragma once

#include <cuda_runtime.h>

#include "aes_kernels.cuh"

namespace paes_b200 {

// Per-device, once: opt the kernels into their dynamic shared memory size.
cudaError_t prepare_kernels();

cudaError_t launch_ecb(bool dec, const EcbArgs& args, int sm_count, cudaStream_t stream);
cudaError_t launch_batch(bool dec, const BatchArgs& args, int sm_count, cudaStream_t stream);
cudaError_t launch_counter_fill(unsigned long long seed, unsigned long long word0, unsigned long long nwords, void* out,
                                int sm_count, cudaStream_t stream);
cudaError_t launch_checksum(const void* buf, unsigned long long nwords, unsigned long long base, unsigned long long* d_out,
                            int sm_count, cudaStream_t stream);
cudaError_t launch_mismatch(const void* a, const void* b, unsigned long long nblocks, unsigned long long* d_out,
                            int sm_count, cudaStream_t stream);
// Single-state round transforms (PAES_OP_*) on n device-resident states.
cudaError_t launch_state_op(int op, std::uint8_t* d_states, unsigned long long n, const StateKey& rk,
                            cudaStream_t stream);
// One 64-bit store on the stream (a result word for an empty transform).
cudaError_t launch_put_u64(unsigned long long* p, unsigned long long v, cudaStream_t stream);
unsigned long long launch_count();

}  // namespace paes_b200
