// tcgen05 (sm_100a) GEMM fast path -- placeholder until the TMEM/TMA kernel lands.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace edpc {
inline bool tc_compiled() { return false; }
inline bool tc_enabled_env() { return false; }
inline bool tc_supported(int, int, int) { return false; }
inline cudaError_t tc_linear_fwd(const float*, int, const float*, int, int, int, const float*,
                                 const float*, float*, int, int64_t, int64_t, cudaStream_t) {
  return cudaErrorNotSupported;
}
}  // namespace edpc
