// Shared helpers for the EDPC B200 kernels: status plumbing, warp reductions.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <string>
#include <utility>

#include "../../include/edpc_b200.h"

namespace edpc {

void set_error(const std::string& msg);

struct Status {
  int code;
};

#define EDPC_CUDA_TRY(expr)                                                          \
  do {                                                                               \
    cudaError_t _e = (expr);                                                         \
    if (_e != cudaSuccess) {                                                         \
      ::edpc::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e) + " @" +  \
                        __FILE__ + ":" + std::to_string(__LINE__));                  \
      return EDPC_ERR_CUDA;                                                          \
    }                                                                                \
  } while (0)

#define EDPC_CHECK_ARG(cond, msg)       \
  do {                                  \
    if (!(cond)) {                      \
      ::edpc::set_error(msg);           \
      return EDPC_ERR_INVALID;          \
    }                                   \
  } while (0)

#define EDPC_TRY(expr)         \
  do {                         \
    int _s = (expr);           \
    if (_s != EDPC_OK) return _s; \
  } while (0)

constexpr int kVocab = 256;
constexpr int kTotal = 1 << 16;
constexpr int kNumGroups = 8;  // fixed lane groups of the G-invariant reduction
// padding of the weight buffers so G <= 8 slices of 64-aligned equal length
// cover them (in-place all-gather of the sharded optimizer's output)
constexpr int64_t kShardPad = kNumGroups * 64;

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Lane-group boundaries of the canonical gradient reduction: group g covers
// global lanes [g*B/8, (g+1)*B/8) (floor division; groups may be empty when B<8).
__host__ __device__ __forceinline__ int group_begin(int g, int B) {
  return (int)(((int64_t)g * B) / kNumGroups);
}

inline int cdiv(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }


// ------------------------------------------------ programmatic dependent launch
//
// Every kernel of a model step is launched with programmatic stream
// serialization (pdl_launch): the next kernel is launched as this one's CTAs
// exit (implicit trigger), runs its prologue, and waits in pdl_entry() for
// the full completion (and memory) of its predecessor -- the launch / ramp
// bubbles between the ~45 kernels of a step overlap (C2: 7.35 -> 7.61 MB/s).
// An explicit early trigger (griddepcontrol.launch_dependents at entry) was
// measured slower (7.05): waiting CTAs then sat on SMs the side-stream
// weight-gradient GEMMs could have used.  A kernel calls pdl_entry() before
// touching anything its predecessor wrote (the tcgen05 GEMM after its TMEM
// allocation).  Without the launch attribute it is a no-op.  EDPC_PDL=0
// disables the attribute.
__device__ __forceinline__ void pdl_entry() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

inline bool pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("EDPC_PDL");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

template <typename... KArgs, typename... Args>
inline cudaError_t pdl_launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace edpc
