// Fused LTE forward (paper dims: F = 256, F' = 64) as ONE kernel instead of
// GEMM -> per-lane FDM -> GEMM.  (A fused backward was built and measured
// slower than up-dgrad + FDM-bwd/Adam + down-dgrad -- 96.9 vs 91.7 us at C2:
// its CTAs ran the projection phases in lockstep and left HBM idle -- and was
// removed.)
//
// Reference: LteBlock.forward / backward (model.py:150-162) = down
// linear_forward (nn.py:78-87), per_row_matmul_forward / _backward
// (nn.py:168-179), up linear_forward; dgrads of linear_backward (nn.py:90-96).
//
// The two projections are tiny (B x 256 x 64 each, 16 K MACs per lane) next to
// the per-lane FDM, which streams each lane's 16 KB matrix U_b (fp32) from HBM
// -- 67 MB per 4096-lane step forward, 402 MB (U, m, v read + written)
// backward.  As separate launches the projections cost more in launch / ramp
// / epilogue latency than in math; here a CTA takes 16 lanes, stages the
// projection weight in shared memory (cp.async, padded rows: conflict-free
// mma fragments), runs the projection on the tensor cores with warp-level
// mma.sync m16n8k8 tf32 (the same tf32 operand precision the tcgen05 path
// uses for these GEMMs), streams the 16 lanes' U rows for the FDM step while
// the second weight is loading, and runs the second projection.  Two CTAs
// per SM (<= 104 KB smem each) keep the U stream going while the other CTA is in
// a projection phase.  The weight-gradient GEMMs of both projections stay on
// the tcgen05 side stream (they reduce over lanes).
#pragma once

#include <cuda_fp16.h>

#include "common.cuh"

namespace edpc {
namespace lte {

constexpr int kRows = 16;         // lanes per CTA
constexpr int kF = 256, kFP = 64;  // feature width, LTE width
constexpr int kThreads = 256;
constexpr int kLdX = kF + 4;       // [16][256] activations: a-fragment rows hit distinct banks
constexpr int kLdS = kFP + 4;      // [16][64] small activations
// weight row strides: b-fragments read (k, n) = W[k][n] (forward, k-major)
// conflict-free with a stride = 8 mod 32, W[n][k] (backward) with 4 mod 32
constexpr int kLdWdF = kFP + 8;    // W_down [256][64], forward
constexpr int kLdWuF = kF + 8;     // W_up [64][256], forward
constexpr int kLdWuB = kF + 4;     // W_up, backward
constexpr int kLdWdB = kFP + 4;    // W_down, backward
constexpr int kWFloats = kF * kLdWdF;  // the largest of the four
static_assert(kWFloats >= kFP * kLdWuF && kWFloats >= kFP * kLdWuB && kWFloats >= kF * kLdWdB);
constexpr int kSmemFloats = kRows * kLdX + kWFloats + 3 * kRows * kLdS;
constexpr size_t kSmemBytes = (size_t)kSmemFloats * 4;
// forward: the weights pass through shared memory in halves (W_down by K rows,
// W_up by N columns) -- 62 KB per CTA, 3 CTAs / SM instead of 2 (ncu: the
// FDM phase was latency-bound at 25% occupancy, r01_ncu_lte_fwd.md).  The
// MMA sequence per output tile is unchanged, so results are bit-identical.
constexpr int kLdWuF2 = kF / 2 + 8;  // W_up column half [64][128]
constexpr int kWFloatsF = (kF / 2) * kLdWdF;
static_assert(kWFloatsF >= kFP * kLdWuF2);
constexpr int kSmemFloatsF = kRows * kLdX + kWFloatsF + 2 * kRows * kLdS;
constexpr size_t kSmemBytesF = (size_t)kSmemFloatsF * 4;

__device__ __forceinline__ void cp_async16(float* smem, const float* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

__device__ __forceinline__ float tf32_round_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__device__ __forceinline__ uint32_t tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t (&a)[4],
                                         const uint32_t (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

// rows x cols fp32 block (global, dense) -> shared (row stride ld), async
__device__ __forceinline__ void stage(float* dst, int ld, const float* src, int rows, int cols) {
  const int c4 = cols / 4;
  for (int e = threadIdx.x; e < rows * c4; e += kThreads) {
    const int r = e / c4, q = e - r * c4;
    cp_async16(dst + r * ld + q * 4, src + (int64_t)r * cols + q * 4);
  }
}

// rows x cols block of a row-major source with row stride src_ld -> shared
__device__ __forceinline__ void stage_ld(float* dst, int ld, const float* src, int src_ld, int rows,
                                        int cols) {
  const int c4 = cols / 4;
  for (int e = threadIdx.x; e < rows * c4; e += kThreads) {
    const int r = e / c4, q = e - r * c4;
    cp_async16(dst + r * ld + q * 4, src + (int64_t)r * src_ld + q * 4);
  }
}

// the CTA's 16 rows of a [Bl][cols] activation (rows past Bl zero-filled)
__device__ __forceinline__ void stage_rows(float* dst, int ld, const float* src, int cols, int b0,
                                           int Bl) {
  const int c4 = cols / 4;
  for (int e = threadIdx.x; e < kRows * c4; e += kThreads) {
    const int r = e / c4, q = e - r * c4;
    if (b0 + r < Bl)
      cp_async16(dst + r * ld + q * 4, src + (int64_t)(b0 + r) * cols + q * 4);
    else
      *reinterpret_cast<float4*>(dst + r * ld + q * 4) = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// acc (one 16 x 8 tile at columns n0..n0+7) += A[16][K] . B, A in smem (row
// stride lda); B element (k, n) at Bs[k * ldb + n] (KMAJ) or Bs[n * ldb + k].
template <int K, bool KMAJ>
__device__ __forceinline__ void warp_tile(float (&acc)[4], const float* As, int lda, const float* Bs,
                                          int ldb, int n0) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll 8
  for (int k0 = 0; k0 < K; k0 += 8) {
    uint32_t a[4], b[2];
    a[0] = tf32(As[g * lda + k0 + t]);
    a[1] = tf32(As[(g + 8) * lda + k0 + t]);
    a[2] = tf32(As[g * lda + k0 + t + 4]);
    a[3] = tf32(As[(g + 8) * lda + k0 + t + 4]);
    if (KMAJ) {
      b[0] = tf32(Bs[(k0 + t) * ldb + n0 + g]);
      b[1] = tf32(Bs[(k0 + t + 4) * ldb + n0 + g]);
    } else {
      b[0] = tf32(Bs[(n0 + g) * ldb + k0 + t]);
      b[1] = tf32(Bs[(n0 + g) * ldb + k0 + t + 4]);
    }
    mma_tf32(acc, a, b);
  }
}

// C fragment rows (g, g + 8), columns (n0 + 2t, n0 + 2t + 1)
struct Frag {
  int r0, c0;
  __device__ Frag(int n0) {
    const int lane = threadIdx.x & 31;
    r0 = lane >> 2;
    c0 = n0 + 2 * (lane & 3);
  }
};

}  // namespace lte

// down = x_local W_d + b_d; mixed_b = down_b U_b; x_lte = mixed W_u + b_u.
// Also stores down and mixed (operands of the FDM backward and of the
// weight-gradient GEMMs).  ln_gain != nullptr: also the global MBRB's layer
// norm of x_lte (nn.py:103-113) -- the x_lte rows of the CTA are complete in
// shared memory here -- with k_embed_ln's arithmetic and element order
// (bit-identical), writing x_hat, rstd and x0 (fp16 x0h, or fp32 x0).
__global__ void __launch_bounds__(lte::kThreads, 3)
k_lte_fwd(const float* __restrict__ x_local, const float* __restrict__ Wd,
          const float* __restrict__ bd, const float* __restrict__ U, const float* __restrict__ Wu,
          const float* __restrict__ bu, float* __restrict__ down, float* __restrict__ mixed,
          float* __restrict__ x_lte, int Bl, const float* __restrict__ ln_gain,
          const float* __restrict__ ln_bias, float* __restrict__ xhat, float* __restrict__ rstd,
          float* __restrict__ x0, __half* __restrict__ x0h, int rt) {
  using namespace lte;
  extern __shared__ float4 lte_smem4[];
  float* Xs = reinterpret_cast<float*>(lte_smem4);
  float* Ws = Xs + kRows * kLdX;
  float* Ds = Ws + kWFloatsF;
  float* Ms = Ds + kRows * kLdS;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int b0 = blockIdx.x * kRows;
  pdl_entry();  // x_local and the weights come from the previous kernels
  stage(Ws, kLdWdF, Wd, kF / 2, kFP);  // W_down rows [0, 128)
  stage_rows(Xs, kLdX, x_local, kF, b0, Bl);
  cp_async_commit();
  cp_async_wait_all();
  __syncthreads();
  {  // down projection: warp w -> columns [8w, 8w + 8), K in two halves
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    warp_tile<kF / 2, true>(acc, Xs, kLdX, Ws, kLdWdF, warp * 8);
    __syncthreads();
    stage(Ws, kLdWdF, Wd + (kF / 2) * kFP, kF / 2, kFP);  // W_down rows [128, 256)
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();
    warp_tile<kF / 2, true>(acc, Xs + kF / 2, kLdX, Ws, kLdWdF, warp * 8);
    const Frag f(warp * 8);
    const float q0 = bd[f.c0], q1 = bd[f.c0 + 1];
    const float2 lo = make_float2(acc[0] + q0, acc[1] + q1), hi = make_float2(acc[2] + q0, acc[3] + q1);
    *reinterpret_cast<float2*>(Ds + f.r0 * kLdS + f.c0) = lo;
    *reinterpret_cast<float2*>(Ds + (f.r0 + 8) * kLdS + f.c0) = hi;
    if (b0 + f.r0 < Bl) *reinterpret_cast<float2*>(down + (int64_t)(b0 + f.r0) * kFP + f.c0) = lo;
    if (b0 + f.r0 + 8 < Bl)
      *reinterpret_cast<float2*>(down + (int64_t)(b0 + f.r0 + 8) * kFP + f.c0) = hi;
  }
  __syncthreads();  // W_d no longer read; down complete
  stage_ld(Ws, kLdWuF2, Wu, kF, kFP, kF / 2);  // W_up columns [0, 128), lands while the FDM step streams U
  cp_async_commit();
  {  // per-lane FDM: 16 threads per lane, float4 columns, 16 rows of U in flight
    const int r = tid >> 4, t = tid & 15, b = b0 + r;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (b < Bl) {
      const float4* u = reinterpret_cast<const float4*>(U + (int64_t)b * kFP * kFP);
      const float* d = Ds + r * kLdS;
#pragma unroll 16
      for (int i = 0; i < kFP; ++i) {
        const float4 q = u[i * (kFP / 4) + t];
        const float di = d[i];
        acc.x = fmaf(di, q.x, acc.x);
        acc.y = fmaf(di, q.y, acc.y);
        acc.z = fmaf(di, q.z, acc.z);
        acc.w = fmaf(di, q.w, acc.w);
      }
      *reinterpret_cast<float4*>(mixed + (int64_t)b * kFP + 4 * t) = acc;
    }
    *reinterpret_cast<float4*>(Ms + r * kLdS + 4 * t) = acc;
  }
  cp_async_wait_all();
  __syncthreads();
#pragma unroll 1
  for (int j = 0; j < kF / 64; ++j) {  // up projection: warp w -> column tiles w, w+8, ...
    if (j == 2) {  // second column half of W_up
      __syncthreads();
      stage_ld(Ws, kLdWuF2, Wu + kF / 2, kF, kFP, kF / 2);
      cp_async_commit();
      cp_async_wait_all();
      __syncthreads();
    }
    const int n0 = (warp + 8 * j) * 8;
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    warp_tile<kFP, true>(acc, Ms, kLdS, Ws + (j >= 2 ? -(kF / 2) : 0), kLdWuF2, n0);
    const Frag f(n0);
    const float q0 = bu[f.c0], q1 = bu[f.c0 + 1];
    const float2 lo = make_float2(acc[0] + q0, acc[1] + q1), hi = make_float2(acc[2] + q0, acc[3] + q1);
    if (b0 + f.r0 < Bl) *reinterpret_cast<float2*>(x_lte + (int64_t)(b0 + f.r0) * kF + f.c0) = lo;
    if (b0 + f.r0 + 8 < Bl)
      *reinterpret_cast<float2*>(x_lte + (int64_t)(b0 + f.r0 + 8) * kF + f.c0) = hi;
    if (ln_gain) {  // the rows for the layer norm below (Xs is free after the down projection)
      *reinterpret_cast<float2*>(Xs + f.r0 * kLdX + f.c0) = lo;
      *reinterpret_cast<float2*>(Xs + (f.r0 + 8) * kLdX + f.c0) = hi;
    }
  }
  if (!ln_gain) return;
  __syncthreads();
  // global-MBRB layer norm: warp w -> rows 2w, 2w+1; lane -> elements lane + 32 j
  const int lane = tid & 31;
#pragma unroll 1
  for (int rr = 0; rr < 2; ++rr) {
    const int r = 2 * warp + rr, b = b0 + r;
    if (b >= Bl) break;
    float v[kF / 32];
#pragma unroll
    for (int j = 0; j < kF / 32; ++j) v[j] = Xs[r * kLdX + lane + 32 * j];
    float sm = 0.f;
#pragma unroll
    for (int j = 0; j < kF / 32; ++j) sm += v[j];
    const float mean = warp_sum(sm) / (float)kF;
    float q = 0.f;
#pragma unroll
    for (int j = 0; j < kF / 32; ++j) {
      const float d = v[j] - mean;
      q += d * d;
    }
    const float var = warp_sum(q) / (float)kF;
    const float rs = 1.0f / sqrtf(var + 1e-5f);
#pragma unroll
    for (int j = 0; j < kF / 32; ++j) {
      const int fidx = lane + 32 * j;
      const float h = (v[j] - mean) * rs;
      xhat[(int64_t)b * kF + fidx] = h;
      const float o = h * ln_gain[fidx] + ln_bias[fidx];
      if (x0h)
        x0h[(int64_t)b * kF + fidx] = __float2half_rn(o);
      else
        x0[(int64_t)b * kF + fidx] = rt ? tf32_round_rna(o) : o;
    }
    if (lane == 0) rstd[b] = rs;
  }
}

}  // namespace edpc
