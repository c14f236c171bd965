// Generic fp32 SIMT GEMM with fused epilogues: the any-shape path.
//
// C[z](m, n) = sum_{s < nsum} sum_{k in K-range} A_s(m, k) * B_s(k, n)
//   A(m,k) = TA ? A[k*lda + m] : A[m*lda + k]
//   B(k,n) = TB ? B[n*ldb + k] : B[k*ldb + n]
// blockIdx.z = zb + nzb * zg: zb selects a batch (pointer strides sA/sB), zg a
// lane group of the canonical gradient reduction (the K range is that
// group's lanes; used by the weight-gradient GEMMs whose K dim is lanes).
//
// The accumulation order is fixed by the tile loop (k ascending in BK
// chunks, s ascending), so results are bitwise reproducible run to run and
// identical between compress and decompress.  This path serves every model
// shape (the reference test-suite's tiny configs included); tc_gemm.cuh is
// the tcgen05 fast path for the paper dims.
#pragma once

#include <stdint.h>

#include "common.cuh"
#include "tc_types.cuh"

namespace edpc {

struct GemmShape {
  int M, N, K;
  const float* A;
  int64_t lda, sA, sA_sum;
  const float* B;
  int64_t ldb, sB, sB_sum;
  int nzb;        // batches
  int nsum;       // summed sub-problems
  // lane-group K split (wgrad): groups [g0, g0 + ngroups) of B_global lanes,
  // local lanes start at global lane `lane0`.  ngroups == 0: K range [0, K).
  int ngroups, g0, B_global, lane0;
};

constexpr int kSimtBM = 64, kSimtBN = 64, kSimtBK = 16;

template <bool TA, bool TB, class Epi>
__global__ void __launch_bounds__(256) k_gemm_simt(GemmShape g, Epi epi) {
  pdl_entry();
  __shared__ float As[kSimtBK][kSimtBM + 4];
  __shared__ float Bs[kSimtBK][kSimtBN + 4];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int m0 = blockIdx.y * kSimtBM, n0 = blockIdx.x * kSimtBN;
  const int zb = blockIdx.z % g.nzb, zg = blockIdx.z / g.nzb;
  int k_begin = 0, k_end = g.K;
  if (g.ngroups > 0) {
    int gg = g.g0 + zg;
    k_begin = group_begin(gg, g.B_global) - g.lane0;
    k_end = group_begin(gg + 1, g.B_global) - g.lane0;
  }
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

  for (int s = 0; s < g.nsum; ++s) {
    const float* A = g.A + zb * g.sA + s * g.sA_sum;
    const float* B = g.B + zb * g.sB + s * g.sB_sum;
    for (int k0 = k_begin; k0 < k_end; k0 += kSimtBK) {
      // A tile: BM x BK (1024 elements, 4 per thread)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        int e = tid + r * 256;
        int mm, kk;
        if (TA) {
          mm = e & (kSimtBM - 1);
          kk = e / kSimtBM;
        } else {
          kk = e & (kSimtBK - 1);
          mm = e / kSimtBK;
        }
        int gm = m0 + mm, gk = k0 + kk;
        float v = 0.f;
        if (gm < g.M && gk < k_end) v = TA ? A[(int64_t)gk * g.lda + gm] : A[(int64_t)gm * g.lda + gk];
        As[kk][mm] = v;
      }
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        int e = tid + r * 256;
        int nn, kk;
        if (TB) {
          kk = e & (kSimtBK - 1);
          nn = e / kSimtBK;
        } else {
          nn = e & (kSimtBN - 1);
          kk = e / kSimtBN;
        }
        int gn = n0 + nn, gk = k0 + kk;
        float v = 0.f;
        if (gn < g.N && gk < k_end) v = TB ? B[(int64_t)gn * g.ldb + gk] : B[(int64_t)gk * g.ldb + gn];
        Bs[kk][nn] = v;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < kSimtBK; ++kk) {
        float a[4], b[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
      }
      __syncthreads();
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int m = m0 + ty + 16 * i;
    if (m >= g.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int n = n0 + tx + 16 * j;
      if (n < g.N) epi(zb, zg, m, n, acc[i][j]);
    }
  }
}

template <bool TA, bool TB, class Epi>
inline cudaError_t gemm_simt(const GemmShape& g, const Epi& epi, cudaStream_t st) {
  int nz = g.nzb * (g.ngroups > 0 ? g.ngroups : 1);
  dim3 grid((unsigned)cdiv(g.N, kSimtBN), (unsigned)cdiv(g.M, kSimtBM), (unsigned)nz);
  if (g.M <= 0 || g.N <= 0 || nz <= 0) return cudaSuccess;
  return pdl_launch(k_gemm_simt<TA, TB, Epi>, grid, dim3(256), 0, st, g, epi);
}

// ------------------------------------------------------------- epilogues
//
// Every epilogue has an element form (SIMT path) and a row32 form (tcgen05
// path: one thread owns 32 consecutive columns of one output row).

__device__ __forceinline__ bool aligned16(const void* p) { return ((uintptr_t)p & 15) == 0; }

__device__ __forceinline__ void load32(const float* src, float (&v)[32]) {
  if (aligned16(src)) {
#pragma unroll
    for (int j = 0; j < 32; j += 4) {
      float4 q = *reinterpret_cast<const float4*>(src + j);
      v[j] = q.x; v[j + 1] = q.y; v[j + 2] = q.z; v[j + 3] = q.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = src[j];
  }
}

__device__ __forceinline__ void store32(float* dst, const float (&v)[32]) {
  if (aligned16(dst)) {
#pragma unroll
    for (int j = 0; j < 32; j += 4)
      *reinterpret_cast<float4*>(dst + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) dst[j] = v[j];
  }
}

// tcgen05 epilogues see a 32x32 block transposed into shared memory:
// T[r * 32 + (j ^ r)] = D(m_base + r, n0 + j); lane j walks the 32 rows of column
// n0 + j, so each warp access is one coalesced 128-byte row segment.
#define EDPC_TILE_ROWS(BODY)                                  \
  {                                                           \
    const int lane_ = threadIdx.x & 31;                       \
    _Pragma("unroll 4") for (int r = 0; r < 32; ++r) {        \
      const int m = m_base + r;                               \
      if (m >= M) break;                                      \
      const float acc = T[r * 32 + (lane_ ^ r)];              \
      BODY                                                    \
    }                                                         \
  }

// C[zb] = acc + bias[zb] (row-broadcast); ldc row stride, sC batch stride
struct EpiBias {
  static constexpr bool kTmaStore = true;
  float* C;
  int64_t ldc, sC;
  const float* bias;
  int64_t sBias;
  bool store_maps(const TcShape& s, TcStoreMap& c, TcStoreMap&) const {
    c = TcStoreMap{C, {(uint64_t)s.N, (uint64_t)s.M, (uint64_t)s.nzb, 1},
                   {(uint64_t)ldc, (uint64_t)sC, 0}};
    return true;
  }
  template <class IO>
  __device__ void ts_chunk(IO& io, int zb, int, int, int n0, float (&v)[1][32]) const {
    float b[32];
    load32(bias + zb * sBias + n0, b);
#pragma unroll
    for (int j = 0; j < 32; ++j) v[0][j] = v[0][j] + b[j];
    io.put(0, v[0], zb, 0);
  }
  __device__ void operator()(int zb, int, int m, int n, float acc) const {
    C[zb * sC + (int64_t)m * ldc + n] = acc + bias[zb * sBias + n];
  }
  __device__ void row32(int zb, int, int m, int n0, float (&v)[32]) const {
    float b[32];
    load32(bias + zb * sBias + n0, b);
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = v[j] + b[j];
    store32(C + zb * sC + (int64_t)m * ldc + n0, v);
  }
  __device__ void tile(const float* T, int zb, int, int m_base, int n0, int M) const {
    const int n = n0 + (threadIdx.x & 31);
    const float b = bias[zb * sBias + n];
    float* Cz = C + zb * sC + n;
    EDPC_TILE_ROWS(Cz[(int64_t)m * ldc] = acc + b;)
  }
};

// C = acc + bias + resid (MBRB out-projection + residual, model.py:102)
struct EpiBiasResid {
  static constexpr bool kTransposed = true;
  float* C;
  int64_t ldc;
  const float* bias;
  const float* resid;
  int64_t ldr;
  int rt = 0;  // output rounded to tf32 (it feeds a tf32 GEMM)
  __device__ float rnd(float x) const {
    if (!rt) return x;
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
  }
  __device__ void operator()(int, int, int m, int n, float acc) const {
    C[(int64_t)m * ldc + n] = rnd((acc + bias[n]) + resid[(int64_t)m * ldr + n]);
  }
  __device__ void row32(int, int, int m, int n0, float (&v)[32]) const {
    float b[32], r[32];
    load32(bias + n0, b);
    load32(resid + (int64_t)m * ldr + n0, r);
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = rnd((v[j] + b[j]) + r[j]);
    store32(C + (int64_t)m * ldc + n0, v);
  }
  __device__ void tile(const float* T, int, int, int m_base, int n0, int M) const {
    const int lane = threadIdx.x & 31;
    const int n = n0 + lane;
    const float b = bias[n];
    const float* __restrict__ R = resid;
    float* __restrict__ O = C;
    float rv[32];
#pragma unroll
    for (int r = 0; r < 32; ++r)
      rv[r] = m_base + r < M ? R[(int64_t)(m_base + r) * ldr + n] : 0.f;
#pragma unroll
    for (int r = 0; r < 32; ++r)
      if (m_base + r < M) O[(int64_t)(m_base + r) * ldc + n] = rnd((T[r * 32 + (lane ^ r)] + b) + rv[r]);
  }
};

// plain store (dgrad outputs)
struct EpiStore {
  static constexpr bool kTmaStore = true;
  float* C;
  int64_t ldc;
  bool store_maps(const TcShape& s, TcStoreMap& c, TcStoreMap&) const {
    c = TcStoreMap{C, {(uint64_t)s.N, (uint64_t)s.M, 1, 1}, {(uint64_t)ldc, 0, 0}};
    return true;
  }
  template <class IO>
  __device__ void ts_chunk(IO& io, int, int, int, int, float (&v)[1][32]) const {
    io.put(0, v[0], 0, 0);
  }
  __device__ void operator()(int, int, int m, int n, float acc) const {
    C[(int64_t)m * ldc + n] = acc;
  }
  __device__ void row32(int, int, int m, int n0, float (&v)[32]) const {
    store32(C + (int64_t)m * ldc + n0, v);
  }
  __device__ void tile(const float* T, int, int, int m_base, int n0, int M) const {
    const int n = n0 + (threadIdx.x & 31);
    EDPC_TILE_ROWS(C[(int64_t)m * ldc + n] = acc;)
  }
};

// plain store plus an fp16 copy (the gradient entering an MBRB: fp32 for the
// LN backward's residual, fp16 as an operand of the fp16 GEMMs)
struct EpiStore2 {
  static constexpr bool kTmaStore = true;
  static constexpr int kTsSlots = 2;
  float* C;
  __half* Ch;
  int64_t ldc;
  bool store_maps(const TcShape& s, TcStoreMap& c, TcStoreMap& d) const {
    c = TcStoreMap{C, {(uint64_t)s.N, (uint64_t)s.M, 1, 1}, {(uint64_t)ldc, 0, 0}};
    d = TcStoreMap{Ch, {(uint64_t)s.N, (uint64_t)s.M, 1, 1}, {(uint64_t)ldc, 0, 0}, 1};
    return true;
  }
  template <class IO>
  __device__ void ts_chunk(IO& io, int, int, int, int, float (&v)[1][32]) const {
    io.put(0, v[0], 0, 0);
    io.put_h(1, v[0], 0, 0);
  }
  __device__ void operator()(int, int, int m, int n, float acc) const {
    C[(int64_t)m * ldc + n] = acc;
    Ch[(int64_t)m * ldc + n] = __float2half_rn(acc);
  }
  __device__ void row32(int, int, int m, int n0, float (&v)[32]) const {
    store32(C + (int64_t)m * ldc + n0, v);
#pragma unroll
    for (int j = 0; j < 32; ++j) Ch[(int64_t)m * ldc + n0 + j] = __float2half_rn(v[j]);
  }
  __device__ void tile(const float* T, int, int, int m_base, int n0, int M) const {
    const int n = n0 + (threadIdx.x & 31);
    EDPC_TILE_ROWS(C[(int64_t)m * ldc + n] = acc; Ch[(int64_t)m * ldc + n] = __float2half_rn(acc);)
  }
};

// weight-gradient partial of lane group (g0 + zg) at param offset (+ zb*sOff)
struct EpiPartial {
  static constexpr bool kTmaStore = true;
  float* partials;     // [8][n_shared]
  int64_t n_shared;
  int64_t off, sOff;   // parameter offset in the shared flat layout, batch stride
  int64_t ldw;         // row stride of the weight (its N)
  int g0;
  bool store_maps(const TcShape& s, TcStoreMap& c, TcStoreMap&) const {
    c = TcStoreMap{partials + off, {(uint64_t)s.N, (uint64_t)s.M, (uint64_t)s.nzb, (uint64_t)kNumGroups},
                   {(uint64_t)ldw, (uint64_t)sOff, (uint64_t)n_shared}};
    return true;
  }
  template <class IO>
  __device__ void ts_chunk(IO& io, int zb, int zg, int, int, float (&v)[1][32]) const {
    io.put(0, v[0], zb, g0 + zg);
  }
  __device__ void operator()(int zb, int zg, int m, int n, float acc) const {
    partials[(int64_t)(g0 + zg) * n_shared + off + zb * sOff + (int64_t)m * ldw + n] = acc;
  }
  __device__ void row32(int zb, int zg, int m, int n0, float (&v)[32]) const {
    store32(partials + (int64_t)(g0 + zg) * n_shared + off + zb * sOff + (int64_t)m * ldw + n0, v);
  }
  __device__ void tile(const float* T, int zb, int zg, int m_base, int n0, int M) const {
    float* P = partials + (int64_t)(g0 + zg) * n_shared + off + zb * sOff + n0 + (threadIdx.x & 31);
    EDPC_TILE_ROWS(P[(int64_t)m * ldw] = acc;)
  }
};

}  // namespace edpc
