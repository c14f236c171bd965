// Types shared by the tcgen05 GEMM (tc_gemm.cuh) and its epilogue functors
// (gemm_simt.cuh, kernels.cuh): the launch shape and the TMA-store output map.
#pragma once

#include <stdint.h>

namespace edpc {

// Where an operand's batch coordinate comes from.
enum TcBatch { kBatchNone = 0, kBatchZ = 1, kBatchSum = 2 };

struct TcShape {
  int M, N, K;       // K per summed sub-problem (before any K split)
  int nzb;           // output batches
  int nsum;          // sub-problems accumulated into one tile
  int a_batch, b_batch;
  // K split, one output per split index zg:
  //   kmode 0: none; 1: lane groups [g0+zg] of B_global lanes (minus lane0);
  //   2: nsplit equal K chunks
  int kmode, nsplit, g0, B_global, lane0;
  int dbg = 0;  // tests only: 1 = epilogue writes m*1000+n; 2/3 = ablations
  int ts = 0;   // set by the launcher: the output tensor map is valid (TMA-store epilogue)
  int mn_lbo = 0, mn_sbo = 0;  // tests only: fp16 MN-major descriptor strides (0 = default)
  // fused column sums of B over K (weight-gradient GEMMs: the bias gradient
  // of lane group g0+zg); needs MN-major B
  float* bias_part = nullptr;
  int64_t bias_gstride = 0, bias_off = 0, bias_zstride = 0;
};

// Output of a TMA-store epilogue as a 4D fp32 tensor: (n, m, c2, c3).
struct TcStoreMap {
  const void* base;
  uint64_t dims[4];     // n (inner), m, c2, c3
  uint64_t strides[3];  // elements, of m, c2, c3
  int half = 0;         // fp16 elements (64B-swizzled 32x32 boxes) instead of fp32
};

}  // namespace edpc
