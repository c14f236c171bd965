// Weight gradient + canonical lane-group tree + Adam in ONE kernel
// (nn.py:90-96 W.grad = X^T dY, model.py:223-235 -> _kernels.py:18-32).
//
// The shared-parameter gradient is the G-invariant tree over 8 fixed lane
// groups, ((g0+g1)+(g2+g3))+((g4+g5)+(g6+g7)).
// The unfused path materialises the 8 group partials in HBM (8 x 19.3 MB per
// step at paper dims) and a separate k_adam_shared re-reads them.  Here a CTA
// owns one 128 x 64 output tile for ALL 8 groups: group g accumulates into its
// own 64-column TMEM slot (8 x 64 = 512 columns), the epilogue drains slot g
// as soon as its K range is done -- folding it into the tree in registers and
// handing the slot back for the next tile -- and after g7 runs Adam on the
// tile with W / m / v TMA-loaded into shared memory and written back (plus
// the fp16 or tf32-rounded shadow the step's GEMMs read) by TMA stores.  The
// bias gradient (column sums of dY, same tree) gets its Adam in the bias
// warps.  Arithmetic is the unfused path's operation for operation -- same
// per-group MMA K order, same tree, same Adam -- so containers are
// bit-identical; what disappears is 2 x 155 MB of partial traffic and the
// Adam launches.  Single context holding all 8 groups only (multi-GPU keeps
// the partials for the slice exchange).
#pragma once

#include "kernels.cuh"
#include "mbrb_fused.cuh"  // tmem_ld16
#include "tc_gemm.cuh"

namespace edpc {

namespace wa {
constexpr int kBN = 64;
constexpr int kStages = 3;
constexpr int kEW = 16;                         // epilogue warps: 4 per TMEM lane quadrant
constexpr int kCW = 16;                         // columns of the 64-wide tile per epilogue warp
constexpr int kStage = (kTcBM + kBN) * 128;     // A 128 rows + B 64 rows of 128-byte K-rows
constexpr int kSlotsPerWarp = 4;                // W, m, v, shadow boxes (32 rows x 16 cols)
constexpr int kBox = 32 * kCW * 4;              // 2 KB
constexpr int kEpi = kEW * kSlotsPerWarp * kBox;
constexpr int kOffEpi = kStages * kStage;
constexpr int kOffBar = kOffEpi + kEpi;
constexpr int kSmemBytes = 1024 + kOffBar + 512;
constexpr int kBiasWarps = 2;                   // 64 columns (fp16: 32 column pairs)
__host__ __device__ constexpr int threads(bool bias) { return 32 * (2 + kEW + (bias ? kBiasWarps : 0)); }
static_assert(kCW * (kEW / 4) == kBN, "epilogue warps cover the tile");
}  // namespace wa

struct WgAdamArgs {
  int Mw, N, nzb;        // output [nzb][Mw][N]
  int B_global, lane0;   // lanes (K) of the 8 groups
  int64_t bias_off, bias_zstride;  // bias parameters (-1: none), relative to W
  float* W;              // fp32 master (M = W + arr, V = W + 2 arr)
  int64_t arr;           // element distance W -> M -> V
  __half* Wh;            // fp16 shadow (H path) or nullptr
  float* Wt;             // tf32-rounded shadow (tf32 path, when rounding) or nullptr
  StepIdx si;
  AdamConsts ac;
  double b1d, b2d;
  float ginv;
  float* keep;           // debug: tree-summed gradient (gradient-scale units) -> here, or nullptr
  int64_t keep_off, keep_ld, keep_zs;
};

// Adam on one fp32 box row (32 values) in shared memory, in place
template <bool H>
__global__ void __launch_bounds__(wa::threads(true), 1)
k_wgrad_adam(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
             const __grid_constant__ CUtensorMap tma_io, const __grid_constant__ CUtensorMap tma_sh,
             WgAdamArgs p, int with_bias) {
  using namespace wa;
  constexpr int BK = tc_bk<H>();
  constexpr int kW = H ? 64 : 32;  // MN width of one TMA box
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kOffBar);
  uint64_t* empty = full + kStages;
  uint64_t* gfull = empty + kStages;   // [8]
  uint64_t* gempty = gfull + 8;        // [8]
  uint64_t* wbar = gempty + 8;         // [kEW] W/m/v boxes of a warp loaded
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(wbar + kEW);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_tn = p.N / kBN, n_tm = (p.Mw + kTcBM - 1) / kTcBM;
  const int n_units = n_tn * n_tm * p.nzb;
  auto coords = [&](int u, int& tn, int& tm, int& zb) {
    tn = u % n_tn;
    tm = (u / n_tn) % n_tm;
    zb = u / (n_tn * n_tm);
  };
  auto krange = [&](int g, int& k0, int& nkb) {
    k0 = group_begin(g, p.B_global) - p.lane0;
    nkb = (group_begin(g + 1, p.B_global) - p.lane0 - k0) / BK;
  };

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tma_a) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tma_b) : "memory");
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], with_bias ? 2 : 1);
    }
    for (int g = 0; g < 8; ++g) {
      mbar_init(&gfull[g], 1);
      mbar_init(&gempty[g], kEW);
    }
    for (int w = 0; w < kEW; ++w) mbar_init(&wbar[w], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_entry();

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer: for each tile, the 8 groups' K ranges
      int it = 0;
      for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        int tn, tm, zb;
        coords(u, tn, tm, zb);
        const int n0 = tn * kBN, m0 = tm * kTcBM;
        for (int g = 0; g < 8; ++g) {
          int k0, nkb;
          krange(g, k0, nkb);
          for (int q = 0; q < nkb; ++q, ++it) {
            const int st = it % kStages;
            mbar_wait(&empty[st], ((uint32_t)(it / kStages) & 1u) ^ 1u);
            uint8_t* sa = smem + st * kStage;
            uint8_t* sb = sa + kTcBM * 128;
            mbar_expect_tx(&full[st], kStage);
            const int k = k0 + q * BK;
#pragma unroll
            for (int j = 0; j < kTcBM / kW; ++j) tma_load_3d(sa + j * kW * 128, &tma_a, &full[st], m0 + kW * j, k, 0);
#pragma unroll
            for (int j = 0; j < kBN / kW; ++j) tma_load_3d(sb + j * kW * 128, &tma_b, &full[st], n0 + kW * j, k, zb);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer: group g -> TMEM slot g
      constexpr uint32_t idesc = H ? idesc_f16(kTcBM, kBN, 1, 1) : idesc_tf32(kTcBM, kBN, 1, 1);
      int it = 0, lu = 0;
      for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++lu) {
        for (int g = 0; g < 8; ++g) {
          int k0, nkb;
          krange(g, k0, nkb);
          mbar_wait_spin(&gempty[g], ((uint32_t)lu & 1u) ^ 1u);
          tc_fence_after();
          const uint32_t d = tmem + (uint32_t)(g * kBN);
          for (int q = 0; q < nkb; ++q, ++it) {
            const int st = it % kStages;
            mbar_wait(&full[st], (uint32_t)(it / kStages) & 1u);
            tc_fence_after();
            const uint32_t sa = smem_u32(smem + st * kStage), sb = sa + kTcBM * 128;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              uint64_t ad, bd;
              if constexpr (H) {
                ad = sdesc(sa + kk * 2048, kMnH_LBO, kMnH_SBO, kLayoutSW128);
                bd = sdesc(sb + kk * 2048, kMnH_LBO, kMnH_SBO, kLayoutSW128);
                tc_mma_f16(d, ad, bd, idesc, (q > 0 || kk > 0) ? 1u : 0u);
              } else {
                ad = sdesc(sa + kk * 1024, 4096, 512, kLayoutSW128Base32B);
                bd = sdesc(sb + kk * 1024, 4096, 512, kLayoutSW128Base32B);
                tc_mma_tf32(d, ad, bd, idesc, (q > 0 || kk > 0) ? 1u : 0u);
              }
            }
            tc_commit(&empty[st]);
          }
          tc_commit(&gfull[g]);
        }
      }
    }
  } else if (warp < 2 + kEW) {
    // ---------------- epilogue: tree over the 8 slots, then Adam on the tile
    // (warp: TMEM lane quadrant `quad`, columns c0 .. c0+15 of the tile)
    const int ew = warp - 2, quad = warp & 3, sub = ew >> 2;
    const int c0 = sub * kCW;
    const uint32_t tq = tmem + ((uint32_t)(quad * 32) << 16);
    float* box = reinterpret_cast<float*>(smem + kOffEpi) + ew * kSlotsPerWarp * (kBox / 4);
    float bc1, bc2;
    adam_bc(p.ac, p.b1d, p.b2d, p.si.T(), bc1, bc2);
    int lu = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++lu) {
      int tn, tm, zb;
      coords(u, tn, tm, zb);
      const int n0 = tn * kBN + c0, mr = tm * kTcBM + quad * 32;
      if (lane == 0) {  // this warp's W / m / v boxes (the previous tile's stores have read them)
        bulk_wait_read<0>();
        mbar_expect_tx(&wbar[ew], 3 * kBox);
        for (int a = 0; a < 3; ++a) tma_load_4d(box + a * (kBox / 4), &tma_io, &wbar[ew], n0, mr, zb, a);
      }
      float acc[kCW], s1[kCW], s2[kCW];  // canonical tree, built as the slots complete
#pragma unroll
      for (int g = 0; g < 8; ++g) {  // unrolled: each step's live set is static
        mbar_wait_spin(&gfull[g], (uint32_t)lu & 1u);
        tc_fence_after();
        float v[kCW];
        tmem_ld16(tq + (uint32_t)(g * kBN + c0), v);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&gempty[g]);
        // ((g0+g1)+(g2+g3)) + ((g4+g5)+(g6+g7))
#pragma unroll
        for (int j = 0; j < kCW; ++j) {
          switch (g) {
            case 0: acc[j] = v[j]; break;
            case 1: acc[j] = acc[j] + v[j]; break;
            case 2: s1[j] = v[j]; break;
            case 3: s1[j] = s1[j] + v[j]; acc[j] = acc[j] + s1[j]; break;
            case 4: s1[j] = v[j]; break;
            case 5: s1[j] = s1[j] + v[j]; break;
            case 6: s2[j] = v[j]; break;
            default: s2[j] = s2[j] + v[j]; s1[j] = s1[j] + s2[j]; acc[j] = acc[j] + s1[j]; break;
          }
        }
      }
      const int m = mr + lane;
      if (p.keep && m < p.Mw) {  // debug: the reduced gradient, as the partial-path slot 0
        float* dst = p.keep + p.keep_off + (int64_t)zb * p.keep_zs + (int64_t)m * p.keep_ld + n0;
        for (int j = 0; j < kCW; ++j) dst[j] = acc[j];
      }
      mbar_wait(&wbar[ew], (uint32_t)lu & 1u);
      // Adam on this thread's row of the 32 x 16 block: fp32 boxes of 64-byte
      // rows (row = lane), 16-byte chunk j at j ^ ((lane >> 1) & 3) (SWIZZLE_64B)
      float* rw = box + lane * kCW;
      float* rm = rw + kBox / 4;
      float* rv = rw + 2 * (kBox / 4);
      float* sh = box + 3 * (kBox / 4);
#pragma unroll
      for (int j4 = 0; j4 < kCW / 4; ++j4) {
        const int o = ((j4 ^ ((lane >> 1) & 3)) << 2);
        float4 w = *reinterpret_cast<float4*>(rw + o);
        float4 mm = *reinterpret_cast<float4*>(rm + o);
        float4 vv = *reinterpret_cast<float4*>(rv + o);
        float* wp = &w.x;
        float* mp = &mm.x;
        float* vp = &vv.x;
#pragma unroll
        for (int e = 0; e < 4; ++e) adam_elem(wp[e], mp[e], vp[e], acc[4 * j4 + e] * p.ginv, p.ac, bc1, bc2);
        *reinterpret_cast<float4*>(rw + o) = w;
        *reinterpret_cast<float4*>(rm + o) = mm;
        *reinterpret_cast<float4*>(rv + o) = vv;
        if constexpr (H) {  // fp16 shadow: rows of 32 B, chunk c at c ^ ((lane >> 2) & 1) (SWIZZLE_32B)
          const int cj = j4 >> 1, hh = j4 & 1;  // 16-byte chunk (8 halves), its 8-byte half
          uint8_t* row = reinterpret_cast<uint8_t*>(sh) + lane * 32;
          __half2 h0 = __floats2half2_rn(w.x, w.y), h1 = __floats2half2_rn(w.z, w.w);
          uint2 q;
          q.x = *reinterpret_cast<uint32_t*>(&h0);
          q.y = *reinterpret_cast<uint32_t*>(&h1);
          *reinterpret_cast<uint2*>(row + ((cj ^ ((lane >> 2) & 1)) << 4) + hh * 8) = q;
        } else {  // tf32-rounded shadow, same layout as W
          *reinterpret_cast<float4*>(sh + lane * kCW + o) =
              make_float4(tf32_rna(w.x), tf32_rna(w.y), tf32_rna(w.z), tf32_rna(w.w));
        }
      }
      fence_async_smem();
      __syncwarp();
      if (lane == 0) {
        for (int a = 0; a < 3; ++a) tma_store_4d(&tma_io, box + a * (kBox / 4), n0, mr, zb, a);
        if (H || p.Wt) tma_store_4d(&tma_sh, sh, n0, mr, zb, 0);
        bulk_commit();
      }
    }
    if (lane == 0) bulk_wait_all();
  } else if (with_bias) {
    // ---------------- bias warps: per-group column sums of dY (the k-block
    // order of the unfused path), the same tree, Adam on the bias entries
    const int bt = threadIdx.x - 32 * (2 + kEW);  // 0..63
    const int n = H ? 2 * bt : bt;                // this thread's column (pair)
    const bool mine = n < kBN;
    float bc1, bc2;
    adam_bc(p.ac, p.b1d, p.b2d, p.si.T(), bc1, bc2);
    int it = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      int tn, tm, zb;
      coords(u, tn, tm, zb);
      const bool do_sum = tm == 0 && p.bias_off >= 0;
      float gs[8], gs2[8];
#pragma unroll
      for (int g = 0; g < 8; ++g) {  // unrolled: gs / gs2 stay in registers
        int k0, nkb;
        krange(g, k0, nkb);
        float sum = 0.f, sum2 = 0.f;
        for (int q = 0; q < nkb; ++q, ++it) {
          const int st = it % kStages;
          mbar_wait(&full[st], (uint32_t)(it / kStages) & 1u);
          if (do_sum && mine) {
            const uint8_t* sb = smem + st * kStage + kTcBM * 128;
            if constexpr (H) {
              const int box = n >> 6, nn = n & 63, chunk = nn >> 3;
              const uint8_t* base = sb + box * 8192 + (nn & 7) * 2;
              float s0 = 0.f, t1 = 0.f;
#pragma unroll 8
              for (int k = 0; k < BK; ++k) {
                const float2 f = __half22float2(*reinterpret_cast<const __half2*>(
                    base + k * 128 + ((chunk ^ (k & 7)) << 4)));
                s0 += f.x;
                t1 += f.y;
              }
              sum += s0;
              sum2 += t1;
            } else {
              const int box = n >> 5, nn = n & 31, chunk = nn >> 3;
              const float* base = reinterpret_cast<const float*>(sb + box * 4096) + (nn & 7);
#pragma unroll 8
              for (int k = 0; k < BK; ++k) sum += base[(k * 128 + ((chunk ^ (k & 3)) << 5)) >> 2];
            }
          }
          named_bar(1, 32 * kBiasWarps);
          if (bt == 0) mbar_arrive(&empty[st]);
        }
        gs[g] = sum;
        gs2[g] = sum2;
      }
      if (do_sum && mine) {
        for (int c = 0; c < (H ? 2 : 1); ++c) {
          const float* q = c ? gs2 : gs;
          const float tree = ((q[0] + q[1]) + (q[2] + q[3])) + ((q[4] + q[5]) + (q[6] + q[7]));
          const int64_t e = p.bias_off + zb * p.bias_zstride + tn * kBN + n + c;
          if (p.keep) p.keep[e] = tree;
          float w = p.W[e], mm = p.W[p.arr + e], vv = p.W[2 * p.arr + e];
          adam_elem(w, mm, vv, tree * p.ginv, p.ac, bc1, bc2);
          p.W[e] = w;
          p.W[p.arr + e] = mm;
          p.W[2 * p.arr + e] = vv;
          if (p.Wh) p.Wh[e] = __float2half_rn(w);
          if (p.Wt) p.Wt[e] = tf32_rna(w);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// 4D map (n, m, z, a) of 32-row x 16-column boxes: fp32 with 64-byte rows
// (SWIZZLE_64B) or fp16 with 32-byte rows (SWIZZLE_32B); element strides of
// m = N, z = sOff, a = sA.  Cached per argument tuple.
inline bool wa_box_map(CUtensorMap* out, const void* base, bool half, int N, int Mw, int nzb, int na,
                       int64_t sOff, int64_t sA) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, bool, int, int, int, int, int64_t, int64_t>, CUtensorMap> cache;
  auto key = std::make_tuple(base, half, N, Mw, nzb, na, sOff, sA);
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find(key);
  if (it != cache.end()) {
    *out = it->second;
    return true;
  }
  const uint64_t es = half ? 2 : 4;
  cuuint64_t dims[4] = {(cuuint64_t)N, (cuuint64_t)Mw, (cuuint64_t)nzb, (cuuint64_t)na};
  cuuint64_t strides[3] = {(cuuint64_t)N * es, (cuuint64_t)(nzb > 1 ? sOff : (int64_t)N * Mw) * es,
                           (cuuint64_t)(na > 1 ? sA : (int64_t)N * Mw * nzb) * es};
  for (auto st : strides)
    if (st % 16 || (uintptr_t)base % 16) return false;
  cuuint32_t box[4] = {16, 32, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  PfnEncodeTiled enc = encode_tiled_fn();
  CUtensorMap m{};
  if (!enc || enc(&m, half ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4,
                  (void*)base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  half ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_64B,
                  CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  cache.emplace(key, m);
  *out = m;
  return true;
}

// Host launcher.  X [lanes][Mw] and G [nzb][lanes][N] (stride sG) are the
// MN-major operands (K = lanes, the 8 lane groups of B_global); the weight is
// W[off + z*sOff + m*N + n] (its bias, if bias_off >= 0, at bias_off +
// z*bias_zstride + n).  io: fp32 4D map over (n, m, z, {W, m, v}); sh: the
// shadow map (fp16 Wh on the H path, tf32-rounded Wt otherwise).
template <bool H>
inline int wgrad_adam_launch(const void* X, int Mw, const void* G, int N, int nzb, int64_t sG,
                             const WgAdamArgs& a0, int64_t off, int64_t sOff, cudaStream_t st) {
  using namespace wa;
  WgAdamArgs a = a0;
  a.Mw = Mw;
  a.N = N;
  a.nzb = nzb;
  TcShape s{Mw, N, a.B_global, nzb, 1, kBatchNone, nzb > 1 ? kBatchZ : kBatchNone, 1, 8, 0,
            a.B_global, a.lane0};
  TcOperand A{X, Mw, 0, 1}, B{G, N, sG, nzb};
  CUtensorMap ta, tb, tio{}, tsh{};
  int r = tc_operand_maps<kBN, true, true, H>(s, A, B, 1, ta, tb);
  if (r != EDPC_OK) return r;
  if (!wa_box_map(&tio, a.W + off, false, N, Mw, nzb, 3, sOff, a.arr) ||
      ((H || a.Wt) && !wa_box_map(&tsh, H ? (const void*)(a.Wh + off) : (const void*)(a.Wt + off),
                                  H, N, Mw, nzb, 1, sOff, 0))) {
    set_error("wgrad_adam: W/m/v or shadow map not encodable (alignment)");
    return EDPC_ERR_INVALID;
  }
  const int with_bias = a.bias_off >= 0 ? 1 : 0;
  static bool attr[16] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr[dev & 15]) {
    cudaFuncSetAttribute(k_wgrad_adam<H>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    attr[dev & 15] = true;
  }
  const int units = (N / kBN) * ((Mw + kTcBM - 1) / kTcBM) * nzb;
  const int grid = units < num_sms() ? units : num_sms();
  cudaError_t e = pdl_launch(k_wgrad_adam<H>, grid, threads(with_bias != 0), kSmemBytes, st, ta, tb,
                             tio, tsh, a, with_bias);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("k_wgrad_adam launch: ") + cudaGetErrorString(e));
    return EDPC_ERR_CUDA;
  }
  return EDPC_OK;
}

}  // namespace edpc

namespace edpc {

// ===================================================================
// Subtree weight gradient: a CTA owns one output tile for HALF of the lane
// groups -- 4 groups, one TMEM slot of BN columns each (4 x BN <= 512) --
// and writes their subtree sum (g0+g1)+(g2+g3) (or the same over g4..g7)
// as ONE partial plane, into partial slot 0 or 4.  The shared Adam then runs
// the top level of the canonical tree over those two slots (NL = 2, stride
// 4 planes): ((g0+g1)+(g2+g3)) + ((g4+g5)+(g6+g7)), bit for bit the 8-leaf
// tree.  Against the per-group partial GEMM: 4x fewer partial planes written
// and read (39 MB instead of 155 MB at paper dims), one wave of CTAs for the
// big weights, each walking 4 groups through a deeper operand ring.
namespace ws {
constexpr int kGpc = 4;         // lane groups per CTA
constexpr int kEW = 16;         // epilogue warps (4 per TMEM lane quadrant)
constexpr int kBiasWarps = 2;
constexpr int kThreads = 32 * (2 + kEW + kBiasWarps);
template <int BN>
struct Geo {
  static constexpr int kCW = BN / (kEW / 4);              // columns per epilogue warp
  static constexpr int kStage = (kTcBM + BN) * 128;       // A + B of one k-block
  static constexpr int kEpi = kEW * 4096;                 // one 32x32 fp32 box per warp
  static constexpr int kStages = (232448 - 2048 - kEpi) / kStage > 6 ? 6 : (232448 - 2048 - kEpi) / kStage;
  static constexpr int kOffEpi = kStages * kStage;
  static constexpr int kOffBar = kOffEpi + kEpi;
  static constexpr int kSmemBytes = 1024 + kOffBar + 512;
};
}  // namespace ws

template <bool H, int BN>
__global__ void __launch_bounds__(ws::kThreads, 1)
k_wgrad_subtree(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                const __grid_constant__ CUtensorMap tma_p, int Mw, int N, int nzb, int B_global,
                int lane0, float* __restrict__ part, int64_t n_shared, int64_t bias_off,
                int64_t bias_zstride, int with_bias) {
  using namespace ws;
  using G = Geo<BN>;
  constexpr int BK = tc_bk<H>();
  constexpr int kW = H ? 64 : 32;
  constexpr int kCW = G::kCW;
  static_assert(kCW == 32 || kCW == 16, "epilogue chunk");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  constexpr int kStages = G::kStages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + G::kOffBar);
  uint64_t* empty = full + kStages;
  uint64_t* gfull = empty + kStages;  // [kGpc]
  uint64_t* gempty = gfull + kGpc;    // [kGpc]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gempty + kGpc);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_tn = N / BN, n_tm = (Mw + kTcBM - 1) / kTcBM;
  const int n_units = n_tn * n_tm * nzb * 2;
  auto coords = [&](int u, int& tn, int& tm, int& zb, int& sub) {
    sub = u & 1;
    const int v = u >> 1;
    tn = v % n_tn;
    tm = (v / n_tn) % n_tm;
    zb = v / (n_tn * n_tm);
  };
  auto krange = [&](int g, int& k0, int& nkb) {
    k0 = group_begin(g, B_global) - lane0;
    nkb = (group_begin(g + 1, B_global) - lane0 - k0) / BK;
  };

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tma_a) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tma_b) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tma_p) : "memory");
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], with_bias ? 2 : 1);
    }
    for (int g = 0; g < kGpc; ++g) {
      mbar_init(&gfull[g], 1);
      mbar_init(&gempty[g], kEW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_entry();

  if (warp == 0) {
    if (lane == 0) {
      int it = 0;
      for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        int tn, tm, zb, sub;
        coords(u, tn, tm, zb, sub);
        const int n0 = tn * BN, m0 = tm * kTcBM;
        for (int gl = 0; gl < kGpc; ++gl) {
          int k0, nkb;
          krange(sub * kGpc + gl, k0, nkb);
          for (int q = 0; q < nkb; ++q, ++it) {
            const int st = it % kStages;
            mbar_wait(&empty[st], ((uint32_t)(it / kStages) & 1u) ^ 1u);
            uint8_t* sa = smem + st * G::kStage;
            uint8_t* sb = sa + kTcBM * 128;
            mbar_expect_tx(&full[st], G::kStage);
            const int k = k0 + q * BK;
#pragma unroll
            for (int j = 0; j < kTcBM / kW; ++j) tma_load_3d(sa + j * kW * 128, &tma_a, &full[st], m0 + kW * j, k, 0);
#pragma unroll
            for (int j = 0; j < BN / kW; ++j) tma_load_3d(sb + j * kW * 128, &tma_b, &full[st], n0 + kW * j, k, zb);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = H ? idesc_f16(kTcBM, BN, 1, 1) : idesc_tf32(kTcBM, BN, 1, 1);
      int it = 0, lu = 0;
      for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++lu) {
        int tn, tm, zb, sub;
        coords(u, tn, tm, zb, sub);
        for (int gl = 0; gl < kGpc; ++gl) {
          int k0, nkb;
          krange(sub * kGpc + gl, k0, nkb);
          mbar_wait_spin(&gempty[gl], ((uint32_t)lu & 1u) ^ 1u);
          tc_fence_after();
          const uint32_t d = tmem + (uint32_t)(gl * BN);
          for (int q = 0; q < nkb; ++q, ++it) {
            const int st = it % kStages;
            mbar_wait(&full[st], (uint32_t)(it / kStages) & 1u);
            tc_fence_after();
            const uint32_t sa = smem_u32(smem + st * G::kStage), sb = sa + kTcBM * 128;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              if constexpr (H) {
                tc_mma_f16(d, sdesc(sa + kk * 2048, kMnH_LBO, kMnH_SBO, kLayoutSW128),
                           sdesc(sb + kk * 2048, kMnH_LBO, kMnH_SBO, kLayoutSW128), idesc,
                           (q > 0 || kk > 0) ? 1u : 0u);
              } else {
                tc_mma_tf32(d, sdesc(sa + kk * 1024, 4096, 512, kLayoutSW128Base32B),
                            sdesc(sb + kk * 1024, 4096, 512, kLayoutSW128Base32B), idesc,
                            (q > 0 || kk > 0) ? 1u : 0u);
              }
            }
            tc_commit(&empty[st]);
          }
          tc_commit(&gfull[gl]);
        }
      }
    }
  } else if (warp < 2 + kEW) {
    // ---------------- epilogue: (q0+q1)+(q2+q3) over the 4 slots -> one partial plane
    const int ew = warp - 2, quad = warp & 3, cw = ew >> 2;
    const int c0 = cw * kCW;
    const uint32_t tq = tmem + ((uint32_t)(quad * 32) << 16);
    float* box = reinterpret_cast<float*>(smem + G::kOffEpi) + ew * 1024;
    int lu = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++lu) {
      int tn, tm, zb, sub;
      coords(u, tn, tm, zb, sub);
      // 16-column passes keep the live set small; the last pass releases the slots
      if (lane == 0) bulk_wait_read<0>();
      __syncwarp();
      // box: 32 rows x kCW fp32 -- 128-byte rows SWIZZLE_128B (kCW 32) or
      // 64-byte rows SWIZZLE_64B (kCW 16)
      float* row = box + lane * kCW;
#pragma unroll
      for (int h = 0; h < kCW / 16; ++h) {
        const bool last = h == kCW / 16 - 1;
        float acc[16], s1[16];
#pragma unroll
        for (int gl = 0; gl < kGpc; ++gl) {
          mbar_wait_spin(&gfull[gl], (uint32_t)lu & 1u);
          tc_fence_after();
          float v[16];
          tmem_ld16(tq + (uint32_t)(gl * BN + c0 + 16 * h), v);
          if (last) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&gempty[gl]);
          }
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            if (gl == 0) acc[j] = v[j];
            else if (gl == 1) acc[j] = acc[j] + v[j];
            else if (gl == 2) s1[j] = v[j];
            else { s1[j] = s1[j] + v[j]; acc[j] = acc[j] + s1[j]; }
          }
        }
#pragma unroll
        for (int j4 = 0; j4 < 4; ++j4) {
          const int ch = kCW == 32 ? ((4 * h + j4) ^ (lane & 7)) : (j4 ^ ((lane >> 1) & 3));
          *reinterpret_cast<float4*>(row + (ch << 2)) =
              make_float4(acc[4 * j4], acc[4 * j4 + 1], acc[4 * j4 + 2], acc[4 * j4 + 3]);
        }
      }
      fence_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_store_4d(&tma_p, box, tn * BN + c0, tm * kTcBM + quad * 32, zb, sub * kGpc);
        bulk_commit();
      }
    }
    if (lane == 0) bulk_wait_all();
  } else if (with_bias) {
    // ---------------- bias warps: the unfused path's per-group column sums, subtree of 4
    const int bt = threadIdx.x - 32 * (2 + kEW);  // 0..63
    int it = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      int tn, tm, zb, sub;
      coords(u, tn, tm, zb, sub);
      const bool do_sum = tm == 0 && bias_off >= 0;
      for (int cb = 0; cb < (H ? BN / 2 : BN); cb += 32 * kBiasWarps) {
        (void)cb;
      }
      constexpr int kCols = (H ? BN / 2 : BN) / (32 * kBiasWarps) > 0 ? (H ? BN / 2 : BN) / (32 * kBiasWarps) : 1;
      float gs[kGpc][kCols], gs2[kGpc][kCols];
#pragma unroll
      for (int gl = 0; gl < kGpc; ++gl) {
        int k0, nkb;
        krange(sub * kGpc + gl, k0, nkb);
        float sum[kCols], sum2[kCols];
#pragma unroll
        for (int j = 0; j < kCols; ++j) sum[j] = sum2[j] = 0.f;
        for (int q = 0; q < nkb; ++q, ++it) {
          const int st = it % kStages;
          mbar_wait(&full[st], (uint32_t)(it / kStages) & 1u);
          if (do_sum) {
            const uint8_t* sb = smem + st * G::kStage + kTcBM * 128;
#pragma unroll
            for (int j = 0; j < kCols; ++j) {
              const int n = H ? 2 * (bt + j * 32 * kBiasWarps) : bt + j * 32 * kBiasWarps;
              if (n < BN) {
                if constexpr (H) {
                  const int bx = n >> 6, nn = n & 63, chunk = nn >> 3;
                  const uint8_t* base = sb + bx * 8192 + (nn & 7) * 2;
                  float s0 = 0.f, t1 = 0.f;
#pragma unroll 8
                  for (int k = 0; k < BK; ++k) {
                    const float2 f = __half22float2(*reinterpret_cast<const __half2*>(
                        base + k * 128 + ((chunk ^ (k & 7)) << 4)));
                    s0 += f.x;
                    t1 += f.y;
                  }
                  sum[j] += s0;
                  sum2[j] += t1;
                } else {
                  const int bx = n >> 5, nn = n & 31, chunk = nn >> 3;
                  const float* base = reinterpret_cast<const float*>(sb + bx * 4096) + (nn & 7);
#pragma unroll 8
                  for (int k = 0; k < BK; ++k) sum[j] += base[(k * 128 + ((chunk ^ (k & 3)) << 5)) >> 2];
                }
              }
            }
          }
          named_bar(1, 32 * kBiasWarps);
          if (bt == 0) mbar_arrive(&empty[st]);
        }
#pragma unroll
        for (int j = 0; j < kCols; ++j) {
          gs[gl][j] = sum[j];
          gs2[gl][j] = sum2[j];
        }
      }
      if (do_sum) {
#pragma unroll
        for (int j = 0; j < kCols; ++j) {
          const int n = H ? 2 * (bt + j * 32 * kBiasWarps) : bt + j * 32 * kBiasWarps;
          float* dst = part + (int64_t)(sub * kGpc) * n_shared + bias_off + zb * bias_zstride + tn * BN + n;
          if (n < BN && tn * BN + n < N) dst[0] = (gs[0][j] + gs[1][j]) + (gs[2][j] + gs[3][j]);
          if (H && n + 1 < BN && tn * BN + n + 1 < N)
            dst[1] = (gs2[0][j] + gs2[1][j]) + (gs2[2][j] + gs2[3][j]);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// Launcher: partials of the weight at `off` (+ z * sOff), row stride N, into
// slots 0 and 4 of part [8][n_shared]; bias (bias_off >= 0) likewise.
template <bool H, int BN>
inline int wgrad_subtree_launch(const void* X, int Mw, const void* G, int N, int nzb, int64_t sG,
                                int B_global, int lane0, float* part, int64_t n_shared, int64_t off,
                                int64_t sOff, int64_t bias_off, cudaStream_t st) {
  using GG = ws::Geo<BN>;
  TcShape s{Mw, N, B_global, nzb, 1, kBatchNone, nzb > 1 ? kBatchZ : kBatchNone, 1, 8, 0, B_global,
            lane0};
  TcOperand A{X, Mw, 0, 1}, B{G, N, sG, nzb};
  CUtensorMap ta, tb, tp;
  int r = tc_operand_maps<BN, true, true, H>(s, A, B, 1, ta, tb);
  if (r != EDPC_OK) return r;
  TcStoreMap pm{part + off, {(uint64_t)N, (uint64_t)Mw, (uint64_t)nzb, (uint64_t)kNumGroups},
                {(uint64_t)N, (uint64_t)sOff, (uint64_t)n_shared}};
  const bool ok = GG::kCW == 32 ? store_tmap_cache().get(&tp, pm)  // 32 x 32 boxes
                                : wa_box_map(&tp, part + off, false, N, Mw, nzb, kNumGroups, sOff,
                                             n_shared);            // 32 x 16 boxes
  if (!ok) {
    set_error("wgrad_subtree: partial map not encodable (alignment)");
    return EDPC_ERR_INVALID;
  }
  static bool attr[16] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr[dev & 15]) {
    cudaFuncSetAttribute(k_wgrad_subtree<H, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         GG::kSmemBytes);
    attr[dev & 15] = true;
  }
  const int units = (N / BN) * ((Mw + kTcBM - 1) / kTcBM) * nzb * 2;
  const int grid = units < num_sms() ? units : num_sms();
  cudaError_t e = pdl_launch(k_wgrad_subtree<H, BN>, grid, ws::kThreads, GG::kSmemBytes, st, ta, tb,
                             tp, Mw, N, nzb, B_global, lane0, part, n_shared, bias_off, sOff,
                             bias_off >= 0 ? 1 : 0);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("k_wgrad_subtree launch: ") + cudaGetErrorString(e));
    return EDPC_ERR_CUDA;
  }
  return EDPC_OK;
}

}  // namespace edpc
