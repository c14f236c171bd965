// Per-step elementwise / per-lane kernels of the EDPC predictor and its online
// update.  Every reduction has a fixed order (warp butterflies, sequential
// lane loops, the 8-group tree), so a step is bitwise reproducible and the
// decoder replays the encoder's trajectory exactly (pkg/src/edpc/__init__.py:1-7).
#pragma once

#include <math_constants.h>
#include <stdint.h>

#include "coder.cuh"
#include "common.cuh"
#include "gemm_simt.cuh"

namespace edpc {

// where a step's context bytes live: row b of the lane matrix, columns
// [i - T, i) are the context (model.py:252-255) and column i the target
struct ByteCols {
  const uint8_t* base;
  int64_t ld;
};

struct StepIdx {
  const int64_t* i;  // current lane column (device)
  const int64_t* t;  // Adam step count (device), model.py:230
  int off;           // steps past (*i, *t): position inside a captured multi-step graph
  __device__ __forceinline__ int64_t I() const { return *i + off; }
  __device__ __forceinline__ int64_t T() const { return *t + off; }
};

// fp32 -> the nearest tf32 value (10-bit mantissa, ties away from zero),
// returned as fp32.  tcgen05 kind::tf32 *truncates* fp32 operands, a bias of
// -2^-12 per operand that does not average out over a K-long dot product
// (measured: max |dp| 3e-3 vs the fp64 oracle on a trained C4a model); GEMM
// operands are therefore stored pre-rounded (numerics bit EDPC_NUM_RND_TF32).
__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// GeLU and its derivative together (_kernels.py:35-51, exact-erf GeLU):
//   GeLU(x) = x Phi(x),  GeLU'(x) = Phi(x) + x phi(x),  Phi(x) = (1 + erf(x/sqrt2)) / 2.
// erf by Abramowitz & Stegun 7.1.26 (|error| <= 1.5e-7), whose e^{-x^2/2}
// factor is phi's too: one ex2 + one rcp for both outputs, ~16 instructions
// against ~35 for erff + expf (ncu: the fused-GeLU GEMM epilogue was issue-
// bound).  Phi is within 3e-7 of the float64 reference over all x.
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float ex2_approx(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ void gelu_pair(float x, float& f, float& dg) {
  const float z = fabsf(x) * 0.70710678118654752f;
  const float t = rcp_approx(fmaf(0.3275911f, z, 1.0f));
  float poly = fmaf(1.061405429f, t, -1.453152027f);
  poly = fmaf(poly, t, 1.421413741f);
  poly = fmaf(poly, t, -0.284496736f);
  poly = fmaf(poly, t, 0.254829592f) * t;
  const float e = ex2_approx((x * -0.72134752044448170f) * x);  // e^{-x^2/2}
  const float half_erf = 0.5f - (0.5f * poly) * e;            // erf(|x|/sqrt2) / 2
  const float cdf = 0.5f + copysignf(half_erf, x);
  f = x * cdf;
  dg = fmaf(x, 0.39894228040143268f * e, cdf);
}

// ------------------------------------------------------ gather + layer norm

constexpr int kLnRowMax = 512;  // rows up to this many features stay in registers

// x = E[ctx] (model.py:255), then LN (nn.py:103-113, population variance,
// eps 1e-5 under the sqrt).  One warp per lane.  gather=false: x is input.
template <bool kGather>
__global__ void __launch_bounds__(256)
k_embed_ln(ByteCols src, StepIdx si, int T, const float* __restrict__ E, int DE, int F, int Bl,
           float* __restrict__ x, const float* __restrict__ gain, const float* __restrict__ bias,
           float* __restrict__ xhat, float* __restrict__ rstd, float* __restrict__ x0,
           __half* __restrict__ x0h, int rt) {
  pdl_entry();
  const int b = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (b >= Bl) return;
  float* xr = x + (int64_t)b * F;
  if (F > kLnRowMax) {  // generic path (rows longer than the register tile)
    float s = 0.f;
    if (kGather) {
      const int64_t col0 = si.I() - T;
      const uint8_t* row = src.base + (int64_t)b * src.ld + col0;
      for (int f = lane; f < F; f += 32) {
        int p = f / DE, d = f - p * DE;
        float v = E[(int)row[p] * DE + d];
        xr[f] = v;
        s += v;
      }
    } else {
      for (int f = lane; f < F; f += 32) s += xr[f];
    }
    const float mean = warp_sum(s) / (float)F;
    float q = 0.f;
    for (int f = lane; f < F; f += 32) {
      float d = xr[f] - mean;
      q += d * d;
    }
    const float var = warp_sum(q) / (float)F;
    const float r = 1.0f / sqrtf(var + 1e-5f);
    for (int f = lane; f < F; f += 32) {
      float h = (xr[f] - mean) * r;
      xhat[(int64_t)b * F + f] = h;
      const float v = h * gain[f] + bias[f];
      if (x0h)
        x0h[(int64_t)b * F + f] = __float2half_rn(v);
      else
        x0[(int64_t)b * F + f] = rt ? tf32_rna(v) : v;
    }
    if (lane == 0) rstd[b] = r;
    return;
  }
  // the row in registers, every gather / load in flight before the sums
  // (re-reading x from global memory made this latency bound)
  constexpr int kJ = kLnRowMax / 32;
  float v[kJ];
  if (kGather) {
    const int64_t col0 = si.I() - T;
    const uint8_t* row = src.base + (int64_t)b * src.ld + col0;
#pragma unroll
    for (int j = 0; j < kJ; ++j) {
      const int f = lane + 32 * j;
      if (f < F) {
        const int p = f / DE, d = f - p * DE;
        v[j] = E[(int)row[p] * DE + d];
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < kJ; ++j)
      if (lane + 32 * j < F) v[j] = xr[lane + 32 * j];
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < kJ; ++j)
    if (lane + 32 * j < F) s += v[j];
  const float mean = warp_sum(s) / (float)F;
  float q = 0.f;
#pragma unroll
  for (int j = 0; j < kJ; ++j)
    if (lane + 32 * j < F) {
      const float d = v[j] - mean;
      q += d * d;
    }
  const float var = warp_sum(q) / (float)F;
  const float r = 1.0f / sqrtf(var + 1e-5f);
#pragma unroll
  for (int j = 0; j < kJ; ++j) {
    const int f = lane + 32 * j;
    if (f < F) {
      if (kGather) xr[f] = v[j];
      const float h = (v[j] - mean) * r;
      xhat[(int64_t)b * F + f] = h;
      const float o = h * gain[f] + bias[f];
      if (x0h)  // fp16 GEMM path: x0 only feeds the branch GEMM and its weight gradient
        x0h[(int64_t)b * F + f] = __float2half_rn(o);
      else  // tf32 GEMM operand: stored rounded to nearest (rt)
        x0[(int64_t)b * F + f] = rt ? tf32_rna(o) : o;
    }
  }
  if (lane == 0) rstd[b] = r;
}

constexpr int kMaxBranches = 8;


// ff = GeLU(prod_z H_z) (model.py:98-101, _kernels.py:35-42).  H_z is then
// overwritten with D_z = GeLU'(prod) * prod_{j != z} H_j, everything the
// backward product rule needs (model.py:107-119): g_H_z = g_ff * D_z.
__global__ void k_mbrb_act(float* __restrict__ H, int K, int64_t plane, float* __restrict__ ff,
                           int rt) {
  pdl_entry();
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= plane) return;
  float h[kMaxBranches];
  float p = H[e];
  h[0] = p;
  for (int z = 1; z < K; ++z) {
    h[z] = H[z * plane + e];
    p = p * h[z];
  }
  float fv, dg;
  gelu_pair(p, fv, dg);
  ff[e] = rt ? tf32_rna(fv) : fv;  // out-projection GEMM operand
  for (int z = 0; z < K; ++z) {
    float d = dg;
    for (int j = 0; j < K; ++j)
      if (j != z) d = d * h[j];
    H[z * plane + e] = d;
  }
}

// MBRB forward epilogue of the multi-branch GEMM (model.py:97-101): H_z =
// acc_z + b_z (kept for the backward product rule), ff = GeLU(prod_z H_z).
template <int ZIN>
struct EpiBranchAct {
  static constexpr bool kTmaStore = true;
  static constexpr int kTsSlots = 2;  // ff and the D_z leave through a 2-box ring
  float* H;         // [ZIN][M][N]
  float* ff;        // [M][N]
  const float* b0;  // bias of branch 0; branch z at b0 + z*sBias
  int64_t sBias, N, plane;
  int rt = 0;       // ff stored rounded to tf32 (it is the out-projection's A operand)
  // map 0: D_z as (n, m, z); map 1: ff
  bool store_maps(const TcShape& s, TcStoreMap& c, TcStoreMap& d) const {
    c = TcStoreMap{H, {(uint64_t)N, (uint64_t)s.M, (uint64_t)ZIN, 1}, {(uint64_t)N, (uint64_t)plane, 0}};
    d = TcStoreMap{ff, {(uint64_t)N, (uint64_t)s.M, 1, 1}, {(uint64_t)N, 0, 0}};
    return true;
  }
  template <class IO>
  __device__ void ts_chunk(IO& io, int, int, int, int n0, float (&v)[ZIN][32]) const {
    float p[32];
#pragma unroll
    for (int z = 0; z < ZIN; ++z) {
      float b[32];
      load32(b0 + z * sBias + n0, b);
#pragma unroll
      for (int j = 0; j < 32; ++j) v[z][j] = v[z][j] + b[j];
#pragma unroll
      for (int j = 0; j < 32; ++j) p[j] = z == 0 ? v[0][j] : p[j] * v[z][j];
    }
    {
      float f[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        gelu_pair(p[j], f[j], p[j]);
        if (rt) f[j] = tf32_rna(f[j]);
      }
      io.put(1, f, 0, 0);
    }
#pragma unroll
    for (int z = 0; z < ZIN; ++z) {
      float d[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        d[j] = p[j];
#pragma unroll
        for (int y = 0; y < ZIN; ++y)
          if (y != z) d[j] = d[j] * v[y][j];
      }
      io.put(0, d, z, 0);
    }
  }
  __device__ void rowz(int m, int n0, float (&v)[ZIN][32]) const {
    float p[32];
#pragma unroll
    for (int z = 0; z < ZIN; ++z) {
      float b[32];
      load32(b0 + z * sBias + n0, b);
#pragma unroll
      for (int j = 0; j < 32; ++j) v[z][j] = v[z][j] + b[j];
#pragma unroll
      for (int j = 0; j < 32; ++j) p[j] = z == 0 ? v[0][j] : p[j] * v[z][j];
    }
    float f[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      gelu_pair(p[j], f[j], p[j]);
      if (rt) f[j] = tf32_rna(f[j]);
    }
    store32(ff + (int64_t)m * N + n0, f);
#pragma unroll
    for (int z = 0; z < ZIN; ++z) {
      float d[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        d[j] = p[j];
#pragma unroll
        for (int y = 0; y < ZIN; ++y)
          if (y != z) d[j] = d[j] * v[y][j];
      }
      store32(H + z * plane + (int64_t)m * N + n0, d);
    }
  }
  __device__ void row32(int, int, int, int, float (&)[32]) const {}
  __device__ void tile(const float*, int, int, int, int, int) const {}
  // T holds ZIN transposed 32x32 blocks (branch z at T + z*32*33).  Stores
  // ff and D_z = GeLU'(prod) * prod_{j != z} H_j (the backward's product-rule
  // factors) -- the backward epilogue is then g_H_z = g_ff * D_z.
  __device__ void tile_z(const float* T, int m_base, int n0, int M) const {
    const int lane = threadIdx.x & 31;
    const int n = n0 + lane;
    float b[ZIN];
#pragma unroll
    for (int z = 0; z < ZIN; ++z) b[z] = b0[z * sBias + n];
#pragma unroll 4
    for (int r = 0; r < 32; ++r) {
      const int m = m_base + r;
      if (m >= M) break;
      const int64_t e = (int64_t)m * N + n;
      float h[ZIN];
      float p = 0.f;
#pragma unroll
      for (int z = 0; z < ZIN; ++z) {
        h[z] = T[z * 1024 + r * 32 + (lane ^ r)] + b[z];
        p = z == 0 ? h[0] : p * h[z];
      }
      float fv, dg;
      gelu_pair(p, fv, dg);
      ff[e] = rt ? tf32_rna(fv) : fv;
#pragma unroll
      for (int z = 0; z < ZIN; ++z) {
        float d = dg;
#pragma unroll
        for (int y = 0; y < ZIN; ++y)
          if (y != z) d = d * h[y];
        H[z * plane + e] = d;
      }
    }
  }
};

// MBRB backward epilogue of the out-projection dgrad (model.py:107-119):
// g_H_z = g_ff * D_z with D_z = GeLU'(prod) * prod_{j != z} H_j stored by
// the forward (k_mbrb_act / EpiBranchAct) in place of H_z.
struct EpiBwdAct {
  static constexpr bool kTransposed = true;  // fallback (K != 2)
  static constexpr bool kTmaStore = true;
  // D_0, D_1 boxes (double-buffered: the next block's load in flight),
  // overwritten in place by g_H_0, g_H_1
  static constexpr int kTsSlots = 4, kTsIn = 2;
  const float* H;  // holds D_z
  float* GH;
  int K;
  int64_t plane, ld;
  // map 0: g_H as (n, m, z); map 1: D as (n, m, z) -- TMA-loaded
  bool store_maps(const TcShape& s, TcStoreMap& c, TcStoreMap& d) const {
    if (K != kTsIn) return false;
    c = TcStoreMap{GH, {(uint64_t)s.N, (uint64_t)s.M, (uint64_t)K, 1}, {(uint64_t)ld, (uint64_t)plane, 0}};
    d = TcStoreMap{H, {(uint64_t)s.N, (uint64_t)s.M, (uint64_t)K, 1}, {(uint64_t)ld, (uint64_t)plane, 0}};
    return true;
  }
  __device__ void ts_in(int i, int, int, int& c2, int& c3) const { c2 = i; c3 = 0; }
  template <class IO>
  __device__ void ts_chunk(IO& io, int, int, int, int, float (&v)[1][32]) const {
#pragma unroll
    for (int z = 0; z < kTsIn; ++z) {
      float d[32];
      io.in(z, d);
#pragma unroll
      for (int j = 0; j < 32; ++j) d[j] = v[0][j] * d[j];
      io.put_at(z, 0, d, z, 0);
    }
  }
  __device__ void operator()(int, int, int m, int n, float acc) const {
    const int64_t e = (int64_t)m * ld + n;
    for (int z = 0; z < K; ++z) GH[z * plane + e] = acc * H[z * plane + e];
  }
  __device__ void row32(int, int, int m, int n0, float (&acc)[32]) const {
    const int64_t e = (int64_t)m * ld + n0;
    for (int z = 0; z < K; ++z) {
      float d[32];
      load32(H + z * plane + e, d);
#pragma unroll
      for (int j = 0; j < 32; ++j) d[j] = acc[j] * d[j];
      store32(GH + z * plane + e, d);
    }
  }
  // all loads of the 32x32 block in flight before the stores
  __device__ void tile(const float* T, int, int, int m_base, int n0, int M) const {
    const int lane = threadIdx.x & 31;
    const int n = n0 + lane;
    const float* __restrict__ Dr = H;
    float* __restrict__ Gw = GH;
    if (K == 2 && m_base + 32 <= M) {
      float d0[32], d1[32];
#pragma unroll
      for (int r = 0; r < 32; ++r) {
        const int64_t e = (int64_t)(m_base + r) * ld + n;
        d0[r] = Dr[e];
        d1[r] = Dr[plane + e];
      }
#pragma unroll
      for (int r = 0; r < 32; ++r) {
        const int64_t e = (int64_t)(m_base + r) * ld + n;
        const float a = T[r * 32 + (lane ^ r)];
        Gw[e] = a * d0[r];
        Gw[plane + e] = a * d1[r];
      }
      return;
    }
    for (int z = 0; z < K; ++z) {
      float d[32];
#pragma unroll
      for (int r = 0; r < 32; ++r)
        d[r] = m_base + r < M ? Dr[z * plane + (int64_t)(m_base + r) * ld + n] : 0.f;
#pragma unroll
      for (int r = 0; r < 32; ++r)
        if (m_base + r < M) Gw[z * plane + (int64_t)(m_base + r) * ld + n] = T[r * 32 + (lane ^ r)] * d[r];
    }
  }
};


// fp16 forms of the two fused MBRB epilogues (the fp16 GEMM path): the same
// math in fp32 registers, ff / D_z / g_H stored as fp16 through 64B-swizzled
// TMA boxes (half the bytes of the fp32 path; 10-bit mantissa = the tf32
// operand precision these values feed).  TMA-only: a launch whose tensor
// maps cannot be built fails instead of taking a fallback.
template <int ZIN>
struct EpiBranchActH {
  static constexpr bool kTmaStore = true, kRequireTs = true;
  // fp16 boxes (2 KB): 4 slots in the 8 KB per warp that 2 fp32 slots took --
  // the 3 stores of a chunk (ff, D_0, D_1) no longer wait on each other
  static constexpr int kTsSlots = 4, kTsSlotBytes = 2048;
  __half* H;        // D_z [ZIN][M][N]
  __half* ff;       // [M][N]
  const float* b0;  // bias of branch 0; branch z at b0 + z*sBias
  int64_t sBias, N, plane;
  int rt = 0;       // ff stored rounded to tf32 (it is the out-projection's A operand)
  bool store_maps(const TcShape& s, TcStoreMap& c, TcStoreMap& d) const {
    c = TcStoreMap{H, {(uint64_t)N, (uint64_t)s.M, (uint64_t)ZIN, 1}, {(uint64_t)N, (uint64_t)plane, 0}, 1};
    d = TcStoreMap{ff, {(uint64_t)N, (uint64_t)s.M, 1, 1}, {(uint64_t)N, 0, 0}, 1};
    return true;
  }
  template <class IO>
  __device__ void ts_chunk(IO& io, int, int, int, int n0, float (&v)[ZIN][32]) const {
    float p[32];
#pragma unroll
    for (int z = 0; z < ZIN; ++z) {
      float b[32];
      load32(b0 + z * sBias + n0, b);
#pragma unroll
      for (int j = 0; j < 32; ++j) v[z][j] = v[z][j] + b[j];
#pragma unroll
      for (int j = 0; j < 32; ++j) p[j] = z == 0 ? v[0][j] : p[j] * v[z][j];
    }
    {
      float f[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) gelu_pair(p[j], f[j], p[j]);
      io.put_h(1, f, 0, 0);
    }
#pragma unroll
    for (int z = 0; z < ZIN; ++z) {
      float d[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        d[j] = p[j];
#pragma unroll
        for (int y = 0; y < ZIN; ++y)
          if (y != z) d[j] = d[j] * v[y][j];
      }
      io.put_h(0, d, z, 0);
    }
  }
  __device__ void row32(int, int, int, int, float (&)[32]) const { __trap(); }
  __device__ void tile(const float*, int, int, int, int, int) const { __trap(); }
  __device__ void tile_z(const float*, int, int, int) const { __trap(); }
};

struct EpiBwdActH {
  static constexpr bool kTmaStore = true, kRequireTs = true;
  static constexpr int kTsSlots = 4, kTsIn = 2, kTsInBytes = 32 * 32 * 2;
  const __half* H;  // D_z
  __half* GH;
  int K;
  int64_t plane, ld;
  bool store_maps(const TcShape& s, TcStoreMap& c, TcStoreMap& d) const {
    if (K != kTsIn) return false;
    c = TcStoreMap{GH, {(uint64_t)s.N, (uint64_t)s.M, (uint64_t)K, 1}, {(uint64_t)ld, (uint64_t)plane, 0}, 1};
    d = TcStoreMap{H, {(uint64_t)s.N, (uint64_t)s.M, (uint64_t)K, 1}, {(uint64_t)ld, (uint64_t)plane, 0}, 1};
    return true;
  }
  __device__ void ts_in(int i, int, int, int& c2, int& c3) const { c2 = i; c3 = 0; }
  template <class IO>
  __device__ void ts_chunk(IO& io, int, int, int, int, float (&v)[1][32]) const {
#pragma unroll
    for (int z = 0; z < kTsIn; ++z) {
      float d[32];
      io.in_h(z, d);
#pragma unroll
      for (int j = 0; j < 32; ++j) d[j] = v[0][j] * d[j];
      io.put_at_h(z, 0, d, z, 0);
    }
  }
  __device__ void operator()(int, int, int, int, float) const { __trap(); }
  __device__ void row32(int, int, int, int, float (&)[32]) const { __trap(); }
  __device__ void tile(const float*, int, int, int, int, int) const { __trap(); }
};

// LN backward + residual (nn.py:116-125, model.py:120-121); one warp per lane
__global__ void __launch_bounds__(256)
k_ln_bwd(const float* __restrict__ gx0, const float* __restrict__ xhat,
         const float* __restrict__ rstd, const float* __restrict__ gain,
         const float* __restrict__ up, float* __restrict__ out, int F, int Bl) {
  pdl_entry();
  const int b = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (b >= Bl) return;
  const int64_t o = (int64_t)b * F;
  float s1 = 0.f, s2 = 0.f;
  for (int f = lane; f < F; f += 32) {
    float g = gx0[o + f] * gain[f];
    s1 += g;
    s2 += g * xhat[o + f];
  }
  const float gm = warp_sum(s1) / (float)F;
  const float gxm = warp_sum(s2) / (float)F;
  const float r = rstd[b];
  for (int f = lane; f < F; f += 32) {
    float g = gx0[o + f] * gain[f];
    out[o + f] = (g - gm - xhat[o + f] * gxm) * r + up[o + f];
  }
}

// LN backward + residual fused with the LN gain / bias gradient partials
// (nn.py:116-125): grid (chunks, groups); a block owns 64 lanes of one lane
// group.  Warps walk lanes w, w+8, ...; each thread keeps column sums of
// gx0 * xhat and gx0 for columns lane, lane+32, ...; warp sums are combined
// in warp order, chunk sums in chunk order by the last block of the group
// (ticket counter) -- a fixed order, so reproducible.
constexpr int kLnChunk = 16;
constexpr int kLnMaxF = 512;

__global__ void __launch_bounds__(256)
k_ln_bwd_fused(const float* __restrict__ gx0, const float* __restrict__ xhat,
               const float* __restrict__ rstd, const float* __restrict__ gain,
               const float* __restrict__ up, float* __restrict__ out, int F, int B_global,
               int lane0, int g0, float* __restrict__ partials, int64_t n_shared, int64_t off_g,
               int64_t off_b, float* __restrict__ scratch, unsigned* __restrict__ tickets) {
  pdl_entry();
  __shared__ float red[8][2 * kLnMaxF];
  __shared__ unsigned ticket;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gg = g0 + blockIdx.y;
  const int gb0 = group_begin(gg, B_global) - lane0, gb1 = group_begin(gg + 1, B_global) - lane0;
  const int lb = gb0 + blockIdx.x * kLnChunk, le = min(gb1, lb + kLnChunk);
  constexpr int kJ = kLnMaxF / 32;
  float sg[kJ], sb[kJ];
#pragma unroll
  for (int j = 0; j < kJ; ++j) sg[j] = sb[j] = 0.f;
  float gn[kJ];
#pragma unroll
  for (int j = 0; j < kJ; ++j) gn[j] = lane + 32 * j < F ? gain[lane + 32 * j] : 0.f;
  // rows b = lb + warp, +8, ... (kLnChunk / 8 = 2 per warp): both rows' loads
  // in flight before the first is used (one DRAM round trip, not two)
  static_assert(kLnChunk == 16, "two rows per warp");
  float gxv2[2][kJ], xhv2[2][kJ], upv2[2][kJ], r2[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int b = lb + warp + 8 * q;
    const int64_t o = (int64_t)b * F;
    r2[q] = b < le ? rstd[b] : 0.f;
#pragma unroll
    for (int j = 0; j < kJ; ++j) {
      const int f = lane + 32 * j;
      const bool ok = b < le && f < F;
      gxv2[q][j] = ok ? gx0[o + f] : 0.f;
      xhv2[q][j] = ok ? xhat[o + f] : 0.f;
      upv2[q][j] = ok ? up[o + f] : 0.f;
    }
  }
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int b = lb + warp + 8 * q;
    if (b >= le) break;
    const int64_t o = (int64_t)b * F;
    const float* gxv = gxv2[q];
    const float* xhv = xhv2[q];
    const float* upv = upv2[q];
    const float r = r2[q];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int j = 0; j < kJ; ++j) {
      if (lane + 32 * j < F) {
        const float g = gxv[j] * gn[j];
        s1 += g;
        s2 += g * xhv[j];
        sg[j] += gxv[j] * xhv[j];
        sb[j] += gxv[j];
      }
    }
    const float gm = warp_sum(s1) / (float)F;
    const float gxm = warp_sum(s2) / (float)F;
#pragma unroll
    for (int j = 0; j < kJ; ++j) {
      const int f = lane + 32 * j;
      if (f < F) out[o + f] = (gxv[j] * gn[j] - gm - xhv[j] * gxm) * r + upv[j];
    }
  }
#pragma unroll
  for (int j = 0; j < kJ; ++j) {
    const int f = lane + 32 * j;
    if (f < F) {
      red[warp][f] = sg[j];
      red[warp][kLnMaxF + f] = sb[j];
    }
  }
  __syncthreads();
  const int nchunk = gridDim.x;
  float* mine = scratch + ((int64_t)blockIdx.y * nchunk + blockIdx.x) * 2 * F;
  for (int f = threadIdx.x; f < F; f += blockDim.x) {
    float a = red[0][f], c = red[0][kLnMaxF + f];
    for (int w = 1; w < 8; ++w) {
      a += red[w][f];
      c += red[w][kLnMaxF + f];
    }
    mine[f] = a;
    mine[F + f] = c;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) ticket = atomicAdd(&tickets[blockIdx.y], 1u);
  __syncthreads();
  if (ticket != (unsigned)(nchunk - 1)) return;
  __threadfence();
  const float* all = scratch + (int64_t)blockIdx.y * nchunk * 2 * F;
  for (int f = threadIdx.x; f < F; f += blockDim.x) {
    // this tail is L2-latency bound: up to 32 chunks' loads issued at once
    // (one round trip), then summed in chunk order
    constexpr int kMaxCh = 32;
    float va[kMaxCh], vc[kMaxCh];
#pragma unroll
    for (int k = 0; k < kMaxCh; ++k) {
      va[k] = k < nchunk ? __ldcg(all + (int64_t)k * 2 * F + f) : 0.f;
      vc[k] = k < nchunk ? __ldcg(all + (int64_t)k * 2 * F + F + f) : 0.f;
    }
    float a = va[0], c = vc[0];
#pragma unroll
    for (int k = 1; k < kMaxCh; ++k)
      if (k < nchunk) {
        a += va[k];
        c += vc[k];
      }
    for (int k = kMaxCh; k < nchunk; ++k) {
      a += __ldcg(all + (int64_t)k * 2 * F + f);
      c += __ldcg(all + (int64_t)k * 2 * F + F + f);
    }
    partials[(int64_t)gg * n_shared + off_g + f] = a;
    partials[(int64_t)gg * n_shared + off_b + f] = c;
  }
  if (threadIdx.x == 0) tickets[blockIdx.y] = 0u;
}

// ------------------------------------------- lane-group column reductions

// partials[g0+zg][off + z*sOff + n] = sum over the group's lanes of
// src[z*sz + b*ld + n] (* mul[b*ld + n] when mul != null): bias and LN
// gradients (nn.py:94, :118-119) as 8 fixed lane-group partials.
// Block = one lane group x 128 columns: warp w sums lanes b0+w, b0+w+8, ...
// (4 columns per thread, float4 when vec), then the 8 warp sums are added in
// warp order -- a fixed tree, so the result is reproducible.
__global__ void __launch_bounds__(256)
k_colsum_groups(const float* __restrict__ src, int64_t ld, int64_t sz,
                const float* __restrict__ mul, int N, float* __restrict__ partials,
                int64_t n_shared, int64_t off, int64_t sOff, int g0, int B_global, int lane0,
                int vec) {
  pdl_entry();
  __shared__ float4 red[8][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = blockIdx.x * 128 + lane * 4;
  const int z = blockIdx.y;
  const int gg = g0 + blockIdx.z;
  const int b0 = group_begin(gg, B_global) - lane0, b1 = group_begin(gg + 1, B_global) - lane0;
  const float* s = src + z * sz;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (n < N) {
#pragma unroll 4
    for (int b = b0 + warp; b < b1; b += 8) {
      const float* row = s + (int64_t)b * ld + n;
      float4 v;
      if (vec) {
        v = *reinterpret_cast<const float4*>(row);
      } else {
        v.x = row[0];
        v.y = n + 1 < N ? row[1] : 0.f;
        v.z = n + 2 < N ? row[2] : 0.f;
        v.w = n + 3 < N ? row[3] : 0.f;
      }
      if (mul) {
        const float* mr = mul + (int64_t)b * ld + n;
        float4 q;
        if (vec) {
          q = *reinterpret_cast<const float4*>(mr);
        } else {
          q.x = mr[0];
          q.y = n + 1 < N ? mr[1] : 0.f;
          q.z = n + 2 < N ? mr[2] : 0.f;
          q.w = n + 3 < N ? mr[3] : 0.f;
        }
        v.x *= q.x; v.y *= q.y; v.z *= q.z; v.w *= q.w;
      }
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  }
  red[warp][lane] = acc;
  __syncthreads();
  if (warp == 0 && n < N) {
    float4 t = red[0][lane];
#pragma unroll
    for (int w = 1; w < 8; ++w) {
      const float4 u = red[w][lane];
      t.x += u.x; t.y += u.y; t.z += u.z; t.w += u.w;
    }
    float* dst = partials + (int64_t)gg * n_shared + off + z * sOff + n;
    dst[0] = t.x;
    if (n + 1 < N) dst[1] = t.y;
    if (n + 2 < N) dst[2] = t.z;
    if (n + 3 < N) dst[3] = t.w;
  }
}

// ---------------------------------------------------- LTE per-lane matrix

// mixed_b = down_b . U_b (nn.py:168-174); one warp per lane
__global__ void __launch_bounds__(256)
k_fdm_fwd(const float* __restrict__ down, const float* __restrict__ U, float* __restrict__ mixed,
          int FP, int Bl, int rt) {
  pdl_entry();
  const int b = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (b >= Bl) return;
  const float* d = down + (int64_t)b * FP;
  const float* u = U + (int64_t)b * FP * FP;
  for (int j = lane; j < FP; j += 32) {
    float acc = 0.f;
    for (int i = 0; i < FP; ++i) acc = fmaf(d[i], u[(int64_t)i * FP + j], acc);
    mixed[(int64_t)b * FP + j] = rt ? tf32_rna(acc) : acc;  // up-projection operand
  }
}

struct AdamConsts {
  float lr, b1, b2, k1, k2, eps;
};

__device__ __forceinline__ double ipow(double a, int64_t e) {
  double r = 1.0;
  while (e) {
    if (e & 1) r *= a;
    e >>= 1;
    a *= a;
  }
  return r;
}

// Per-launch Adam constants from the bias corrections bc1 = 1 - b1^t,
// bc2 = 1 - b2^t (t shared by all parameters, numba's exponentiation by
// squaring): step = lr / bc1 and rs2 = 1 / sqrt(bc2).
__device__ __forceinline__ void adam_bc(const AdamConsts& c, double b1d, double b2d, int64_t t,
                                        float& step, float& rs2) {
  const double bc1 = 1.0 - ipow(b1d, t), bc2 = 1.0 - ipow(b2d, t);
  step = (float)((double)c.lr / bc1);
  rs2 = (float)(1.0 / sqrt(bc2));
}

// _kernels.py:26-31 in fp32: w -= lr * (m/bc1) / (sqrt(v/bc2) + eps), with the
// bias corrections folded into the per-launch constants and one fast division
// (~2 ulp; it scales the update, not w) instead of two IEEE divisions and a
// sqrt of a quotient -- the per-lane FDM Adam was issue-bound on them.
__device__ __forceinline__ void adam_elem(float& w, float& m, float& v, float g,
                                          const AdamConsts& c, float step, float rs2) {
  const float mi = c.b1 * m + c.k1 * g;
  const float vi = c.b2 * v + c.k2 * (g * g);
  m = mi;
  v = vi;
  w -= __fdividef(step * mi, fmaf(sqrtf(vi), rs2, c.eps));
}

// Fused FDM backward + per-lane Adam (nn.py:177-179 then _kernels.py:18-32 on
// lane_mats): g_down_b = g_mixed_b . U_b^T with the pre-update U, then
// U_b -= Adam(down_b (x) g_mixed_b).  U, m, v are read and written once.
__global__ void __launch_bounds__(256)
k_fdm_bwd_adam(const float* __restrict__ down, const float* __restrict__ gmix,
               float* __restrict__ U, float* __restrict__ Um, float* __restrict__ Uv,
               float* __restrict__ gdown, int FP, int Bl, StepIdx si, AdamConsts c, double b1d,
               double b2d, float ginv) {
  pdl_entry();
  const int b = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (b >= Bl) return;
  float bc1, bc2;
  adam_bc(c, b1d, b2d, si.T(), bc1, bc2);
  const float* d = down + (int64_t)b * FP;
  const float* gm = gmix + (int64_t)b * FP;
  const int64_t base = (int64_t)b * FP * FP;
  for (int i = 0; i < FP; ++i) {
    float acc = 0.f;
    const float di = d[i] * ginv;  // gradient scale removed exactly (see k_dlogits)
    for (int j = lane; j < FP; j += 32) {
      const int64_t e = base + (int64_t)i * FP + j;
      float w = U[e], m = Um[e], v = Uv[e];
      const float gj = gm[j];
      acc = fmaf(gj, w, acc);
      adam_elem(w, m, v, di * gj, c, bc1, bc2);
      U[e] = w;
      Um[e] = m;
      Uv[e] = v;
    }
    acc = warp_sum(acc);
    if (lane == 0) gdown[(int64_t)b * FP + i] = acc;
  }
}

// ------------------------------------ vectorised FDM kernels (F' = 64/128/256)
//
// kTPR threads own one row of U_b (float4 each, kNV per thread); a warp
// covers 32/kTPR lanes at once.  Row-dot reductions use xor shuffles within
// the kTPR-thread group (fixed tree -> reproducible).

template <int FP>
struct FdmGeo {
  static constexpr int kTPR = FP / 4 < 32 ? FP / 4 : 32;
  static constexpr int kNV = FP / (4 * kTPR);
  static constexpr int kLPW = 32 / kTPR;  // lanes (matrices) per warp
};

template <int FP>
__global__ void __launch_bounds__(256)
k_fdm_fwd_v(const float* __restrict__ down, const float* __restrict__ U, float* __restrict__ mixed,
            int Bl, int rt) {
  pdl_entry();
  using G = FdmGeo<FP>;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int b = warp * G::kLPW + lane / G::kTPR;
  const int t = lane % G::kTPR;
  if (b >= Bl) return;
  const float* d = down + (int64_t)b * FP;
  const float4* u = reinterpret_cast<const float4*>(U + (int64_t)b * FP * FP);
  float4 acc[G::kNV];
#pragma unroll
  for (int v = 0; v < G::kNV; ++v) acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 16  // 16 rows of U in flight per thread
  for (int i = 0; i < FP; ++i) {
    const float di = d[i];
#pragma unroll
    for (int v = 0; v < G::kNV; ++v) {
      const float4 q = u[(i * FP) / 4 + v * G::kTPR + t];
      acc[v].x = fmaf(di, q.x, acc[v].x);
      acc[v].y = fmaf(di, q.y, acc[v].y);
      acc[v].z = fmaf(di, q.z, acc[v].z);
      acc[v].w = fmaf(di, q.w, acc[v].w);
    }
  }
  float4* out = reinterpret_cast<float4*>(mixed + (int64_t)b * FP);
#pragma unroll
  for (int v = 0; v < G::kNV; ++v) {
    if (rt) {  // up-projection operand
      acc[v].x = tf32_rna(acc[v].x); acc[v].y = tf32_rna(acc[v].y);
      acc[v].z = tf32_rna(acc[v].z); acc[v].w = tf32_rna(acc[v].w);
    }
    out[v * G::kTPR + t] = acc[v];
  }
}

// GX: g_down_b = U_b g_b with the old U (nn.py:177-179); ADAM: U_b's
// gradient d_b (x) g_b and its Adam step.  Both in one pass (U read once),
// or split so that the Adam half -- ~6 B/param of HBM traffic, off the
// critical path -- runs on the side stream after the GX half.
template <int FP, bool GX = true, bool ADAM = true>
__global__ void __launch_bounds__(256)
k_fdm_bwd_adam_v(const float* __restrict__ down, const float* __restrict__ gmix,
                 float* __restrict__ U, float* __restrict__ Um, float* __restrict__ Uv,
                 float* __restrict__ gdown, int Bl, StepIdx si, AdamConsts c, double b1d,
                 double b2d, float ginv) {
  pdl_entry();
  using G = FdmGeo<FP>;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int b = warp * G::kLPW + lane / G::kTPR;
  const int t = lane % G::kTPR;
  const bool live = b < Bl;
  const int bb = live ? b : 0;
  float bc1 = 0.f, bc2 = 0.f;
  if (ADAM) adam_bc(c, b1d, b2d, si.T(), bc1, bc2);
  const float* d = down + (int64_t)bb * FP;
  const float4* gm4 = reinterpret_cast<const float4*>(gmix + (int64_t)bb * FP);
  float4 g[G::kNV];
#pragma unroll
  for (int v = 0; v < G::kNV; ++v) g[v] = gm4[v * G::kTPR + t];
  float4* u4 = reinterpret_cast<float4*>(U + (int64_t)bb * FP * FP);
  float4* m4 = reinterpret_cast<float4*>(Um + (int64_t)bb * FP * FP);
  float4* v4 = reinterpret_cast<float4*>(Uv + (int64_t)bb * FP * FP);
  // rows in batches of 8: all 24 float4 loads of a batch are in flight
  // before the Adam math; the 8 row-dot reductions follow the stores
  constexpr int kR = 8;
#pragma unroll 1
  for (int i0 = 0; i0 < FP; i0 += kR) {
    float4 w[kR][G::kNV], m[kR][G::kNV], q[kR][G::kNV];
#pragma unroll
    for (int r = 0; r < kR; ++r)
#pragma unroll
      for (int v = 0; v < G::kNV; ++v) {
        const int e = ((i0 + r) * FP) / 4 + v * G::kTPR + t;
        w[r][v] = u4[e];
        if (ADAM) {
          m[r][v] = m4[e];
          q[r][v] = v4[e];
        }
      }
    float part[kR];
#pragma unroll
    for (int r = 0; r < kR; ++r) {
      const float di = ADAM ? d[i0 + r] * ginv : 0.f;  // (d ginv) g == d (g ginv): exact
      part[r] = 0.f;
#pragma unroll
      for (int v = 0; v < G::kNV; ++v) {
        if (GX) {
          part[r] = fmaf(g[v].x, w[r][v].x, part[r]);
          part[r] = fmaf(g[v].y, w[r][v].y, part[r]);
          part[r] = fmaf(g[v].z, w[r][v].z, part[r]);
          part[r] = fmaf(g[v].w, w[r][v].w, part[r]);
        }
        if (ADAM) {
          adam_elem(w[r][v].x, m[r][v].x, q[r][v].x, di * g[v].x, c, bc1, bc2);
          adam_elem(w[r][v].y, m[r][v].y, q[r][v].y, di * g[v].y, c, bc1, bc2);
          adam_elem(w[r][v].z, m[r][v].z, q[r][v].z, di * g[v].z, c, bc1, bc2);
          adam_elem(w[r][v].w, m[r][v].w, q[r][v].w, di * g[v].w, c, bc1, bc2);
          if (live) {
            const int e = ((i0 + r) * FP) / 4 + v * G::kTPR + t;
            u4[e] = w[r][v];
            m4[e] = m[r][v];
            v4[e] = q[r][v];
          }
        }
      }
    }
    if (GX) {
#pragma unroll
      for (int r = 0; r < kR; ++r) {
#pragma unroll
        for (int o = G::kTPR / 2; o > 0; o >>= 1)
          part[r] += __shfl_xor_sync(0xffffffffu, part[r], o);
        if (live && t == 0) gdown[(int64_t)b * FP + i0 + r] = part[r];
      }
    }
  }
}

// ------------------------------------------------ embedding scatter-add

// Deterministic replacement of np.add.at (model.py:276-278).  Each chunk is
// <= 16 consecutive lanes of one lane group (<= 4096 context bytes); the
// chunk's context bytes and gradient rows are staged in shared memory, then
// thread c (= byte value) walks the (lane, position) entries in order and
// accumulates the matching rows.  chunk_tab[k] = {group, lane begin, end}.
constexpr int kEmbChunkLanes = 16;
constexpr int kEmbSmemFloats = 4096;  // 16 KB of gradient rows per chunk

// Block-local stable counting sort of the chunk's (lane, position) entries
// by context byte: histogram (int atomics: order-free) -> exclusive scan ->
// stable ranks from __match_any_sync + per-warp counts.  Thread c then sums
// exactly its byte's rows in entry order -- the same order as a sequential
// scan, so results do not depend on scheduling.
__global__ void __launch_bounds__(256)
k_embed_grad_chunks(ByteCols src, StepIdx si, int T, int DE, int F,
                    const float* __restrict__ gx, const int* __restrict__ chunk_tab,
                    float* __restrict__ sub) {
  pdl_entry();
  __shared__ uint8_t cbytes[4096];
  __shared__ float grows[kEmbSmemFloats];
  __shared__ int hist[256], off[256], run[256];
  __shared__ int wcnt[8][256];
  __shared__ short order[4096];
  const int k = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int lb = chunk_tab[3 * k + 1], le = chunk_tab[3 * k + 2];
  const int nl = le - lb;
  const int n = nl * T;
  const int64_t col0 = si.I() - T;
  for (int e = tid; e < n; e += blockDim.x) {
    int bl = e / T, p = e - bl * T;
    cbytes[e] = src.base[(int64_t)(lb + bl) * src.ld + col0 + p];
  }
  const bool staged = nl * F <= kEmbSmemFloats;
  if (staged) {  // float4, 4 loads in flight per thread (an LDG->STS chain was latency bound)
    const float4* g0 = reinterpret_cast<const float4*>(gx + (int64_t)lb * F);
    float4* gr = reinterpret_cast<float4*>(grows);
    const int n4 = (nl * F) >> 2;
    if (((nl * F) & 3) == 0 && (((uintptr_t)g0) & 15) == 0) {
      for (int e0 = tid; e0 < n4; e0 += 4 * blockDim.x) {
        float4 q[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (e0 + u * (int)blockDim.x < n4) q[u] = g0[e0 + u * blockDim.x];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (e0 + u * (int)blockDim.x < n4) gr[e0 + u * blockDim.x] = q[u];
      }
    } else {
      for (int e = tid; e < nl * F; e += blockDim.x) grows[e] = gx[(int64_t)lb * F + e];
    }
  }
  hist[tid] = 0;
  __syncthreads();
  for (int e = tid; e < n; e += blockDim.x) atomicAdd(&hist[cbytes[e]], 1);
  __syncthreads();
  // exclusive scan of hist (256 entries, one per thread): warp scans + totals
  {
    const int h = hist[tid];
    int incl = h;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) wcnt[0][warp] = incl;
    __syncthreads();
    int before = 0;
    for (int w = 0; w < warp; ++w) before += wcnt[0][w];
    off[tid] = before + incl - h;
    run[tid] = before + incl - h;
  }
  __syncthreads();
  // stable positions, 256 entries per pass
  for (int t0 = 0; t0 < n; t0 += 256) {
    const int e = t0 + tid;
    const bool live = e < n;
    const int b = live ? cbytes[e] : 256 + lane;  // distinct dummies never match real bytes
    const unsigned same = __match_any_sync(0xffffffffu, b);
    const int lrank = __popc(same & ((1u << lane) - 1u));
    for (int q = tid; q < 8 * 256; q += blockDim.x) (&wcnt[0][0])[q] = 0;
    __syncthreads();
    if (live && lrank == 0) wcnt[warp][b] = __popc(same);
    __syncthreads();
    if (live) {
      int r = run[b] + lrank;
      for (int w = 0; w < warp; ++w) r += wcnt[w][b];
      order[r] = (short)e;
    }
    __syncthreads();
    {  // advance the running per-byte counters past this pass
      int add = 0;
      for (int w = 0; w < 8; ++w) add += wcnt[w][tid];
      run[tid] += add;
    }
    __syncthreads();
  }
  // half-warp per byte value, thread = embedding dimension: the 16 threads
  // read one row's 16 consecutive floats (conflict-free; a thread per byte
  // value reading whole rows hit 2 banks, ~16-way conflicts) and sum the
  // byte's entries in their sorted (= sequential scan) order
  const int hw = tid >> 4, dl = tid & 15;
  for (int c = hw; c < 256; c += 16) {
    const int o0 = off[c], o1 = off[c] + hist[c];
    for (int d = dl; d < ((DE + 15) & ~15); d += 16) {
      float acc = 0.f;
      if (d < DE) {
        for (int q = o0; q < o1; ++q) {
          const int e = order[q];
          const int bl = e / T, p = e - bl * T;
          acc += staged ? grows[bl * F + p * DE + d] : gx[(int64_t)(lb + bl) * F + p * DE + d];
        }
        sub[((int64_t)k * 256 + c) * DE + d] = acc;
      }
    }
  }
}

// group partial = sum of its chunks, in chunk order
__global__ void k_embed_grad_reduce(const float* __restrict__ sub, const int* __restrict__ grp_chunks,
                                    int DE, float* __restrict__ partials, int64_t n_shared,
                                    int64_t off) {
  pdl_entry();
  const int gl = blockIdx.y;  // local group slot
  const int gg = grp_chunks[3 * gl], k0 = grp_chunks[3 * gl + 1], k1 = grp_chunks[3 * gl + 2];
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= 256 * DE) return;
  float acc = 0.f;
#pragma unroll 8
  for (int k = k0; k < k1; ++k) acc += sub[(int64_t)k * 256 * DE + e];
  partials[(int64_t)gg * n_shared + off + e] = acc;
}

// ------------------------------------------------------- fp16 helpers

__global__ void k_to_tf32(const float* __restrict__ src, float* __restrict__ dst, int64_t n) {
  pdl_entry();
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    dst[e] = tf32_rna(src[e]);
}

__global__ void k_to_half(const float* __restrict__ src, __half* __restrict__ dst, int64_t n) {
  pdl_entry();
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    dst[e] = __float2half_rn(src[e]);
}

// ------------------------------------------------------- Adam (shared)

// Pairwise tree over NL in {1,2,4,8} leaves q[0..NL): for NL = 8 this is
// ((q0+q1)+(q2+q3))+((q4+q5)+(q6+q7)) -- the canonical G-invariant order over
// the 8 lane groups.  A subtree of 8/G consecutive groups is
// itself a tree of this shape, so "subtree sums on each of G ranks, then the
// NL = G tree over the subtree sums" is bit-identical to the NL = 8 tree.
template <int NL>
__device__ __forceinline__ float tree_sum(const float* q) {
  if constexpr (NL == 1) {
    return q[0];
  } else {
    return tree_sum<NL / 2>(q) + tree_sum<NL / 2>(q + NL / 2);
  }
}

// grad = tree over NL leaves (leaf g of param e at P[g * pstride + e]) then
// fused Adam (_kernels.py:18-32).  NL = 8: the 8 lane-group partials of one
// context; NL = G: the G ranks' subtree sums of this rank's owned slice
// (multi-GPU, after the slice exchange).
template <int NL>
__global__ void k_adam_shared(float* __restrict__ W, float* __restrict__ M, float* __restrict__ V,
                              const float* __restrict__ P, int64_t n, int64_t pstride, StepIdx si,
                              AdamConsts c, double b1d, double b2d, float ginv,
                              __half* __restrict__ Wh, float* __restrict__ Wt) {
  pdl_entry();
  float bc1, bc2;
  adam_bc(c, b1d, b2d, si.T(), bc1, bc2);
  int64_t head = 0;
  // 16-byte vectors when every stream is aligned (same per-element
  // arithmetic, so bit-identical); the scalar loop takes the tail
  const bool vec = ((((uintptr_t)W | (uintptr_t)M | (uintptr_t)V | (uintptr_t)P |
                      (uintptr_t)Wt) & 15) == 0) &&
                   (pstride & 3) == 0 && ((uintptr_t)Wh & 7) == 0;
  if (vec) {
    const int64_t n4 = n >> 2;
    for (int64_t e4 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e4 < n4;
         e4 += (int64_t)gridDim.x * blockDim.x) {
      float4 q4[NL];
#pragma unroll
      for (int g = 0; g < NL; ++g) q4[g] = reinterpret_cast<const float4*>(P + g * pstride)[e4];
      float4 w4 = reinterpret_cast<const float4*>(W)[e4];
      float4 m4 = reinterpret_cast<const float4*>(M)[e4];
      float4 v4 = reinterpret_cast<const float4*>(V)[e4];
      float* wv = &w4.x;
      float* mv = &m4.x;
      float* vv = &v4.x;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float q[NL];
#pragma unroll
        for (int g = 0; g < NL; ++g) q[g] = (&q4[g].x)[j];
        const float grad = tree_sum<NL>(q) * ginv;
        adam_elem(wv[j], mv[j], vv[j], grad, c, bc1, bc2);
      }
      reinterpret_cast<float4*>(W)[e4] = w4;
      reinterpret_cast<float4*>(M)[e4] = m4;
      reinterpret_cast<float4*>(V)[e4] = v4;
      if (Wh) {
        __half2 h0 = __floats2half2_rn(w4.x, w4.y), h1 = __floats2half2_rn(w4.z, w4.w);
        uint2 hh;
        hh.x = *reinterpret_cast<uint32_t*>(&h0);
        hh.y = *reinterpret_cast<uint32_t*>(&h1);
        reinterpret_cast<uint2*>(Wh)[e4] = hh;
      }
      if (Wt)
        reinterpret_cast<float4*>(Wt)[e4] =
            make_float4(tf32_rna(w4.x), tf32_rna(w4.y), tf32_rna(w4.z), tf32_rna(w4.w));
    }
    head = n4 << 2;
  }
  for (int64_t e = head + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    float q[NL];
#pragma unroll
    for (int g = 0; g < NL; ++g) q[g] = P[g * pstride + e];
    const float grad = tree_sum<NL>(q) * ginv;
    float w = W[e], m = M[e], v = V[e];
    adam_elem(w, m, v, grad, c, bc1, bc2);
    W[e] = w;
    if (Wh) Wh[e] = __float2half_rn(w);  // fp16 shadow for the fp16 GEMMs
    if (Wt) Wt[e] = tf32_rna(w);         // tf32-rounded shadow for the tf32 GEMMs
    M[e] = m;
    V[e] = v;
  }
}

// Multi-GPU: P[0][e] = tree over this rank's NL lane-group partials
// P[g * pstride + e] (in place into leaf 0; elementwise, so no hazard).
template <int NL>
__global__ void k_group_tree(float* __restrict__ P, int64_t n, int64_t pstride) {
  pdl_entry();
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    float q[NL];
#pragma unroll
    for (int g = 0; g < NL; ++g) q[g] = P[g * pstride + e];
    P[e] = tree_sum<NL>(q);
  }
}

// --------------------------------------------------- softmax + quantizer

enum QuantMode { kProbsOnly = 0, kEncode = 1, kDecode = 2 };

// nn.py:186-190 softmax in fp32, then the quantizer on the exact doubles of
// the fp32 probabilities (coder.py:58-80).  kEncode writes the target
// symbol's (cum_lo | freq << 16) into intervals[i][b]; kDecode writes the
// row's cumulative table (cum[0..255] as u16; cum[256] = 65536 implied).
template <int kMode>
__global__ void __launch_bounds__(256)
k_softmax_quant(const float* __restrict__ logits, float* __restrict__ probs, int Bl,
                ByteCols src, StepIdx si, uint32_t* __restrict__ intervals,
                uint16_t* __restrict__ cdf16, float Bf, float gscale, float* __restrict__ g) {
  pdl_entry();
  const int b = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (b >= Bl) return;
  const float* lg = logits + (int64_t)b * 256 + lane * 8;
  float x[8];
  float4 v0 = *reinterpret_cast<const float4*>(lg);
  float4 v1 = *reinterpret_cast<const float4*>(lg + 4);
  x[0] = v0.x; x[1] = v0.y; x[2] = v0.z; x[3] = v0.w;
  x[4] = v1.x; x[5] = v1.y; x[6] = v1.z; x[7] = v1.w;
  float mx = x[0];
#pragma unroll
  for (int j = 1; j < 8; ++j) mx = fmaxf(mx, x[j]);
  mx = warp_max(mx);
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    x[j] = expf(x[j] - mx);
    s += x[j];
  }
  s = warp_sum(s);
  double p[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    x[j] = x[j] / s;
    p[j] = (double)x[j];
  }
  float* pr = probs + (int64_t)b * 256 + lane * 8;
  *reinterpret_cast<float4*>(pr) = make_float4(x[0], x[1], x[2], x[3]);
  *reinterpret_cast<float4*>(pr + 4) = make_float4(x[4], x[5], x[6], x[7]);
  if (kMode == kProbsOnly) return;
  int freq[8];
  warp_quantize<false>(p, freq);
  uint32_t cum[8];
  warp_cdf(freq, cum);
  const int64_t i = si.I();
  if (kMode == kEncode) {
    const int tgt = src.base[(int64_t)b * src.ld + i];
    if (g) {  // the loss gradient, fused (k_dlogits' exact arithmetic; the target is known)
      float gv[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) gv[j] = ((lane * 8 + j == tgt ? x[j] - 1.0f : x[j]) / Bf) * gscale;
      float* gr = g + (int64_t)b * 256 + lane * 8;
      *reinterpret_cast<float4*>(gr) = make_float4(gv[0], gv[1], gv[2], gv[3]);
      *reinterpret_cast<float4*>(gr + 4) = make_float4(gv[4], gv[5], gv[6], gv[7]);
    }
    if ((tgt >> 3) == lane) {
      uint32_t lo = 0, fr = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if ((tgt & 7) == j) {
          lo = cum[j];
          fr = (uint32_t)freq[j];
        }
      intervals[i * Bl + b] = lo | (fr << 16);
    }
  } else {
    uint16_t* dst = cdf16 + (int64_t)b * 256 + lane * 8;
    uint4 pk;
    pk.x = cum[0] | (cum[1] << 16);
    pk.y = cum[2] | (cum[3] << 16);
    pk.z = cum[4] | (cum[5] << 16);
    pk.w = cum[6] | (cum[7] << 16);
    *reinterpret_cast<uint4*>(dst) = pk;
  }
}

// dlogits = (probs - onehot(target)) / B (nn.py:204-210); nll for the loss
// The gradient leaves scaled by gscale = 2^k (k = floor(log2 B)): |g| <= 1,
// so fp16 GEMM operands do not underflow; every backward op is linear in g
// and power-of-two scaling commutes with fp32 rounding, and the Adam kernels
// multiply by 1/gscale, so the fp32 trajectory is bit-identical to unscaled.
__global__ void k_dlogits(const float* __restrict__ probs, ByteCols src, StepIdx si, int Bl,
                          float Bf, float gscale, float* __restrict__ g, float* __restrict__ nll) {
  pdl_entry();
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)Bl * 256) return;
  const int b = (int)(e >> 8), v = (int)(e & 255);
  const int tgt = src.base[(int64_t)b * src.ld + si.I()];
  float p = probs[e];
  if (v == tgt) {
    if (nll) nll[b] = -logf(p);
    p = p - 1.0f;
  }
  g[e] = (p / Bf) * gscale;
}

// --------------------------------------------------------------- coder

// bootstrap intervals: the first min(t, L) columns under the uniform table
// (pipeline.py:84-90, coder.py:118-123)
__global__ void k_boot_intervals(const uint8_t* __restrict__ mat, int64_t L, int Bl, int64_t ncols,
                                 uint32_t* __restrict__ intervals) {
  pdl_entry();
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= ncols * Bl) return;
  const int64_t i = e / Bl;
  const int b = (int)(e - i * Bl);
  const uint32_t s = mat[(int64_t)b * L + i];
  intervals[e] = (s * 256u) | (256u << 16);
}

// Stage B of DPCA on the device: one thread per segment walks lane columns
// [i0, i1) and its lanes in order (pipeline.py:152-153, 182-184).
__global__ void k_encode_columns(const uint32_t* __restrict__ intervals, int Bl, int spl, int Sl,
                                 int64_t i0, int64_t i1, int64_t* __restrict__ enc_state,
                                 uint32_t* __restrict__ words, int64_t cap_words) {
  pdl_entry();
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= Sl) return;
  int64_t* stp = enc_state + 4 * s;
  EncState st{(uint64_t)stp[0], (uint64_t)stp[1], (uint64_t)stp[2], (uint64_t)stp[3]};
  BitWriter w;
  w.open(words + (int64_t)s * cap_words, st.bitpos, (uint64_t)cap_words);
  const int b0 = s * spl;
  for (int64_t i = i0; i < i1; ++i) {
    const uint32_t* row = intervals + i * Bl + b0;
    for (int b = 0; b < spl; ++b) {
      const uint32_t iv = row[b];
      const uint32_t lo = iv & 0xffffu;
      enc_symbol(st, w, lo, lo + (iv >> 16));
    }
  }
  w.close();
  stp[0] = (int64_t)st.low;
  stp[1] = (int64_t)st.high;
  stp[2] = (int64_t)st.pending;
  stp[3] = (int64_t)w.bitpos;
}

__global__ void k_encode_finish_all(int64_t* __restrict__ enc_state, uint32_t* __restrict__ words,
                                    int64_t cap_words, int Sl) {
  pdl_entry();
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= Sl) return;
  int64_t* stp = enc_state + 4 * s;
  EncState st{(uint64_t)stp[0], (uint64_t)stp[1], (uint64_t)stp[2], (uint64_t)stp[3]};
  BitWriter w;
  w.open(words + (int64_t)s * cap_words, st.bitpos, (uint64_t)cap_words);
  enc_finish(st, w);
  w.close();
  stp[2] = 0;
  stp[3] = (int64_t)w.bitpos;
}

// Container assembly on the device: segment s's finished
// bitstream (its bytes, in stream order, at words + s * cap_words) is copied to
// out + off[s], so the whole payload area of the container leaves the GPU in
// one D2H copy instead of one per segment.  One block per segment.
__global__ void k_pack_payloads(const uint32_t* __restrict__ words, int64_t cap_words,
                                const int64_t* __restrict__ off, uint8_t* __restrict__ out, int Sl) {
  pdl_entry();
  const int s = blockIdx.x;
  if (s >= Sl) return;
  const uint8_t* src = reinterpret_cast<const uint8_t*>(words + (int64_t)s * cap_words);
  const int64_t o = off[s], nb = off[s + 1] - o;
  for (int64_t k = threadIdx.x; k < nb; k += blockDim.x) out[o + k] = src[k];
}

__global__ void k_decoder_init_all(int64_t* __restrict__ dec_state, const uint8_t* __restrict__ pay,
                                   const int64_t* __restrict__ pay_off,
                                   const int64_t* __restrict__ bits, int Sl) {
  pdl_entry();
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= Sl) return;
  const uint8_t* d = pay + pay_off[s];
  uint64_t code = 0;
  for (int k = 0; k < 32; ++k) code = (code << 1) | read_bit(d, bits[s], k);
  int64_t* stp = dec_state + 4 * s;
  stp[0] = 0;
  stp[1] = (int64_t)kMask32;
  stp[2] = (int64_t)code;
  stp[3] = 32;
}

// One warp per segment decodes lane column i for its lanes (pipeline.py:272-275);
// uniform=true is the bootstrap table.  On exhaustion the segment's error
// flag is set and its remaining symbols decode as 0 (host raises CoderError).
__global__ void k_decode_column(uint8_t* __restrict__ mat, int64_t L, StepIdx si, int spl, int Sl,
                                const uint16_t* __restrict__ cdf16, bool uniform,
                                int64_t* __restrict__ dec_state, const uint8_t* __restrict__ pay,
                                const int64_t* __restrict__ pay_off,
                                const int64_t* __restrict__ bits, int* __restrict__ err) {
  pdl_entry();
  const int s = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (s >= Sl) return;
  const int64_t i = si.I();
  int64_t* stp = dec_state + 4 * s;
  const bool dead = err[s] != 0;
  DecState st{(uint64_t)stp[0], (uint64_t)stp[1], (uint64_t)stp[2], stp[3]};
  const uint8_t* data = pay + pay_off[s];
  const int64_t nbits = bits[s];
  bool ok = !dead;
  // the segment's CDF rows are independent of the coder state: loaded kPf
  // rows ahead (double-buffered) so the serial symbol chain never waits on them
  constexpr int kPf = 8;
  uint4 cur[kPf], nxt[kPf];
  auto load_rows = [&](uint4 (&q)[kPf], int bl0) {
#pragma unroll
    for (int j = 0; j < kPf; ++j)
      if (!uniform && bl0 + j < spl)
        q[j] = *reinterpret_cast<const uint4*>(cdf16 + (int64_t)(s * spl + bl0 + j) * 256 + lane * 8);
  };
  load_rows(cur, 0);
  for (int g0 = 0; g0 < spl; g0 += kPf) {
    if (g0 + kPf < spl) load_rows(nxt, g0 + kPf);
#pragma unroll
    for (int j = 0; j < kPf; ++j) {
      const int bl = g0 + j;
      if (bl >= spl) break;
      const int b = s * spl + bl;
      int sym = 0;
      if (ok) {
        uint32_t cum[8];
        if (uniform) {
#pragma unroll
          for (int u = 0; u < 8; ++u) cum[u] = (uint32_t)(lane * 8 + u) * 256u;
        } else {
          const uint4 pk = cur[j];
          cum[0] = pk.x & 0xffffu; cum[1] = pk.x >> 16;
          cum[2] = pk.y & 0xffffu; cum[3] = pk.y >> 16;
          cum[4] = pk.z & 0xffffu; cum[5] = pk.z >> 16;
          cum[6] = pk.w & 0xffffu; cum[7] = pk.w >> 16;
        }
        const uint64_t span = st.high - st.low + 1;
        const uint64_t value = dec_value(st, span);
        uint32_t c_lo, c_hi;
        sym = warp_find_symbol(cum, value, c_lo, c_hi);
        ok = dec_advance(st, data, nbits, span, c_lo, c_hi);
        if (!ok) sym = 0;
      }
      if (lane == 0) mat[(int64_t)b * L + i] = (uint8_t)sym;
    }
#pragma unroll
    for (int j = 0; j < kPf; ++j) cur[j] = nxt[j];
  }
  if (lane == 0) {
    if (!ok && !dead) err[s] = 1;
    stp[0] = (int64_t)st.low;
    stp[1] = (int64_t)st.high;
    stp[2] = (int64_t)st.code;
    stp[3] = st.bitpos;
  }
}

// Split-K epilogue: tile partial of K chunk zg into the workspace.
struct EpiSplit {
  static constexpr bool kTmaStore = true;
  float* ws;
  int64_t ld, plane;
  bool store_maps(const TcShape& s, TcStoreMap& c, TcStoreMap&) const {
    c = TcStoreMap{ws, {(uint64_t)s.N, (uint64_t)s.M, (uint64_t)s.nsplit, 1},
                   {(uint64_t)ld, (uint64_t)plane, 0}};
    return true;
  }
  template <class IO>
  __device__ void ts_chunk(IO& io, int, int zg, int, int, float (&v)[1][32]) const {
    io.put(0, v[0], zg, 0);
  }
  __device__ void operator()(int, int zg, int m, int n, float acc) const {
    ws[zg * plane + (int64_t)m * ld + n] = acc;
  }
  __device__ void row32(int, int zg, int m, int n0, float (&v)[32]) const {
    store32(ws + zg * plane + (int64_t)m * ld + n0, v);
  }
  __device__ void tile(const float* T, int, int zg, int m_base, int n0, int M) const {
    float* W = ws + zg * plane + n0 + (threadIdx.x & 31);
    EDPC_TILE_ROWS(W[(int64_t)m * ld] = acc;)
  }
};

// out = ((ws0 + ws1) + ws2) + ... (fixed order) then (+ bias) (+ resid):
// the reduction of a split-K GEMM, fused with its bias/residual epilogue.
__global__ void k_splitk_reduce(const float* __restrict__ ws, int nsplit, int64_t plane, int N,
                                const float* __restrict__ bias, const float* __restrict__ resid,
                                float* __restrict__ out, int rt) {
  pdl_entry();
  const int64_t e = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (e >= plane) return;
  // every load issued before the first add (a dependent loop kept one in flight)
  constexpr int kMax = 4;
  float4 w[kMax];
#pragma unroll
  for (int s = 0; s < kMax; ++s)
    if (s < nsplit) w[s] = *reinterpret_cast<const float4*>(ws + s * plane + e);
  const int n = (int)(e % N);
  const float4 b = bias ? *reinterpret_cast<const float4*>(bias + n) : make_float4(0.f, 0.f, 0.f, 0.f);
  const float4 r = resid ? *reinterpret_cast<const float4*>(resid + e) : make_float4(0.f, 0.f, 0.f, 0.f);
  float4 a = w[0];
#pragma unroll
  for (int s = 1; s < kMax; ++s)
    if (s < nsplit) {
      a.x += w[s].x; a.y += w[s].y; a.z += w[s].z; a.w += w[s].w;
    }
  for (int s = kMax; s < nsplit; ++s) {
    const float4 q = *reinterpret_cast<const float4*>(ws + s * plane + e);
    a.x += q.x; a.y += q.y; a.z += q.z; a.w += q.w;
  }
  if (bias) {
    a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
  }
  if (resid) {
    a.x += r.x; a.y += r.y; a.z += r.z; a.w += r.w;
  }
  if (rt) {  // the MBRB output feeds a tf32 GEMM (LTE down-projection / head)
    a.x = tf32_rna(a.x); a.y = tf32_rna(a.y); a.z = tf32_rna(a.z); a.w = tf32_rna(a.w);
  }
  *reinterpret_cast<float4*>(out + e) = a;
}

__global__ void k_step_advance(int64_t* i, int64_t* t, int n) {
  pdl_entry();
  *i += n;
  *t += n;
}

}  // namespace edpc
