// Fused MBRB forward (model.py:95-103) on the tcgen05 tensor cores: the two
// branch GEMMs, the product / GeLU epilogue and the out-projection GEMM in one
// kernel, the hidden tile never leaving the SM between the two GEMMs.
//
//   H_z  = x0 . W_z + b_z        (z = 0, 1; x0 = LN(x), fp16 [Bl][F])
//   ff   = GeLU(H_0 * H_1)       (stored fp16: the out-proj weight gradient)
//   D_z  = GeLU'(H_0 H_1) H_{1-z} (stored fp16: the backward's product rule)
//   part[s] = ff[:, hs] . W_out[hs, :]   over the CTA's slice hs of H
//
// A CTA owns one 128-row tile of lanes and one of kFusedSplit equal slices of
// the hidden dimension H, walked in chunks of kHC = 64 columns:
//   warp 0       TMA producer: x0 tile once (resident, 64 KB), per chunk the
//                two branch-weight boxes of each 64-deep k-block (ring of
//                kB1Stages), running ahead of the epilogue
//   warp 2+kEW   TMA producer of the chunk's 64 x 256 out-projection weight
//                rows (its own thread, so the branch-weight ring never waits
//                behind the out-projection's buffer)
//   warp 1       TMEM allocation + MMA1 issuer (one thread):
//                  MMA1(c): acc1[c & 1][z] = x0 . W_z[:, chunk c]   (both
//                           branches in one N = 128 instruction), issued as
//                           soon as the epilogue has loaded acc1[c & 1] of
//                           chunk c-2 (acc1 double-buffered in TMEM)
//   warp 4+kEW   MMA2 issuer (one thread): acc2 += ff(c) . W_out[chunk c, :]
//                (N = 256) once the epilogue has staged ff(c)
//   warp 3+kEW   store warp: TMA-stores each chunk's staged ff / D_z tiles and
//                hands the staging back (mbarriers, no CTA-wide barriers)
//   warps 2..    kEW = 16 epilogue warps (4 per TMEM lane quadrant, 16 columns
//                of a chunk each): tcgen05.ld of both branches (acc1 released right
//                after the load), bias / product / GeLU / GeLU', then ff into
//                the shared-memory A operand of MMA2 (K-major, 128B swizzle)
//                and D_z into staging tiles, which the store warp copies out.  After the last chunk the 128 x 256
//                fp32 accumulator acc2 goes to the split-K workspace; the
//                existing k_splitk_reduce adds the slices in a fixed order
//                with bias and residual -- done in the kernel: the kFusedSplit
//                CTAs of a row tile are one thread-block cluster and sum their
//                partials over distributed shared memory in rank order.
// TMEM: acc1 2 x 2 x 64 columns + acc2 256 columns = 512.
//
// The arithmetic is the unfused path's, operation for operation: the branch
// GEMM accumulates K = F in 16-deep steps, the epilogue is EpiBranchActH's,
// the out-projection accumulates each H slice in the same 16-deep steps as the
// kFusedSplit-way split-K GEMM it replaces, and the slices are reduced by the
// same kernel -- so the containers are bit-identical to the unfused path.
#pragma once

#include "kernels.cuh"
#include "tc_gemm.cuh"

namespace edpc {

namespace mf {
constexpr int kBM = 128;
constexpr int kF = 256;          // feature width (x0 row, out-projection N)
constexpr int kHC = 64;          // hidden chunk
constexpr int kB1Stages = 4;
constexpr int kMaxSlice = 1024;  // hidden columns per CTA whose branch biases sit in smem
constexpr int kPrefetch = 2;     // chunks of weights prefetched into L2 ahead of the ring
constexpr int kEW = 16;          // epilogue warps (kEW / 4 per TMEM lane quadrant)
constexpr int kCW = kHC / (kEW / 4);  // columns of a chunk per epilogue warp
// + the out-projection weight producer, the store warp and the MMA2 issuer
constexpr int kThreads = 32 * (2 + kEW + 3);
constexpr int kA1Bytes = kBM * kF * 2;             // 64 KB resident x0 tile
constexpr int kB1Stage = 2 * kHC * 64 * 2;          // both branches, one 64-deep k-block: 16 KB
constexpr int kB2Bytes = kHC * kF * 2;              // 32 KB
constexpr int kA2Bytes = kBM * kHC * 2;             // 16 KB
constexpr int kDBytes = 2 * kBM * kHC * 2;          // 32 KB (D_0, D_1)
constexpr int kOffA1 = 0;
constexpr int kOffB1 = kOffA1 + kA1Bytes;
constexpr int kOffB2 = kOffB1 + kB1Stages * kB1Stage;
constexpr int kOffA2 = kOffB2 + kB2Bytes;
constexpr int kOffD = kOffA2 + kA2Bytes;
constexpr int kOffBias = kOffD + kDBytes;              // [2][kMaxSlice] fp32
constexpr int kOffBar = kOffBias + 2 * kMaxSlice * 4;
constexpr int kSmemBytes = 1024 + kOffBar + 256;
}  // namespace mf

constexpr int kFusedSplit = 4;  // = kSplitK of the unfused out-projection

// L2 prefetch of a TMA box (no shared memory, no completion tracking)
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* map, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(map),
               "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}

__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1,
                                             int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(map),
      "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// 32 lanes x 16 consecutive fp32 TMEM columns -> 16 registers per thread
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
}

template <int N>
__device__ __forceinline__ void tmem_ldn(uint32_t taddr, float (&v)[N]) {
  if constexpr (N == 32)
    tmem_ld32(taddr, v);
  else
    tmem_ld16(taddr, v);
}

// N fp32 values -> fp16, into 2N bytes of a K-major SWIZZLE_128B row (row r
// of a 128-byte-row tile): 16-byte chunk j (8 halves) at (j ^ (r & 7)).
template <int N>
__device__ __forceinline__ void put_row_h_sw128(uint8_t* tile, int r, int j0, const float (&v)[N]) {
  const uint32_t row = smem_u32(tile) + (uint32_t)(r * 128);
#pragma unroll
  for (int jj = 0; jj < N / 8; ++jj) {
    __half2 h0 = __floats2half2_rn(v[8 * jj], v[8 * jj + 1]);
    __half2 h1 = __floats2half2_rn(v[8 * jj + 2], v[8 * jj + 3]);
    __half2 h2 = __floats2half2_rn(v[8 * jj + 4], v[8 * jj + 5]);
    __half2 h3 = __floats2half2_rn(v[8 * jj + 6], v[8 * jj + 7]);
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(
                     row + (uint32_t)(((j0 + jj) ^ (r & 7)) << 4)),
                 "r"(*reinterpret_cast<uint32_t*>(&h0)), "r"(*reinterpret_cast<uint32_t*>(&h1)),
                 "r"(*reinterpret_cast<uint32_t*>(&h2)), "r"(*reinterpret_cast<uint32_t*>(&h3))
                 : "memory");
  }
}

// grid: (ceil(Bl / 128) * kFusedSplit); tile t = blockIdx.x / kFusedSplit,
// slice s = blockIdx.x % kFusedSplit
__global__ void __launch_bounds__(mf::kThreads, 1)
k_mbrb_fwd_fused(const __grid_constant__ CUtensorMap tm_x0, const __grid_constant__ CUtensorMap tm_wb,
                 const __grid_constant__ CUtensorMap tm_wo, const __grid_constant__ CUtensorMap tm_ff,
                 const __grid_constant__ CUtensorMap tm_d, const float* __restrict__ b0,
                 int64_t sBias, int Bl, int H, const float* __restrict__ bias_out,
                 const float* __restrict__ resid, float* __restrict__ out, int rt) {
  using namespace mf;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA1 = smem + kOffA1;
  uint8_t* sB1 = smem + kOffB1;
  uint8_t* sB2 = smem + kOffB2;
  uint8_t* sA2 = smem + kOffA2;
  uint8_t* sD = smem + kOffD;
  float* sBiasT = reinterpret_cast<float*>(smem + kOffBias);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + kOffBar);
  uint64_t* a1full = bar;
  uint64_t* b1full = bar + 1;
  uint64_t* b1empty = b1full + kB1Stages;
  uint64_t* b2full = b1empty + kB1Stages;  // [2] out-projection weight halves (n 0-127, 128-255)
  uint64_t* b2empty = b2full + 2;          // [2]
  uint64_t* tfull1 = b2empty + 2;   // [2]
  uint64_t* tempty1 = tfull1 + 2;   // [2]
  uint64_t* staged = tempty1 + 2;   // ff / D_z of a chunk written (one arrive per epilogue warp)
  uint64_t* a2empty = staged + 1;   // MMA2 done reading ff
  uint64_t* sfree = a2empty + 1;    // the chunk's TMA stores done reading the staging tiles
  uint64_t* t2full = sfree + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(t2full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x / kFusedSplit, split = blockIdx.x % kFusedSplit;
  const int m0 = tile * kBM;
  const int hs = H / kFusedSplit;           // hidden columns of this slice
  const int h_begin = split * hs;
  const int nc = hs / kHC;                  // chunks

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_x0) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_wb) : "memory");
    mbar_init(a1full, 1);
    for (int s = 0; s < kB1Stages; ++s) {
      mbar_init(&b1full[s], 1);
      mbar_init(&b1empty[s], 1);
    }
    for (int q = 0; q < 2; ++q) {
      mbar_init(&b2full[q], 1);
      mbar_init(&b2empty[q], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull1[b], 1);
      mbar_init(&tempty1[b], kEW);
    }
    mbar_init(staged, kEW);
    mbar_init(a2empty, 1);
    mbar_init(sfree, 1);
    mbar_init(t2full, 1);
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
  if (warp == 0 && lane == 0) {  // weights into L2 while the predecessor drains
    for (int c = 0; c < kPrefetch && c < nc; ++c) {
      for (int kb = 0; kb < kF / 64; ++kb)
        for (int z = 0; z < 2; ++z) tma_prefetch_3d(&tm_wb, h_begin + c * kHC, kb * 64, z);
      for (int j = 0; j < kF / 64; ++j) tma_prefetch_3d(&tm_wo, j * 64, h_begin + c * kHC, 0);
    }
  }
  pdl_entry();

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer
      mbar_expect_tx(a1full, kA1Bytes);
#pragma unroll
      for (int kb = 0; kb < kF / 64; ++kb) tma_load_3d(sA1 + kb * 16384, &tm_x0, a1full, kb * 64, m0, 0);
      int it = 0;
      for (int c = 0; c < nc; ++c) {
        const int h0 = h_begin + c * kHC;
        if (c + kPrefetch < nc)  // the ring's source, kPrefetch chunks ahead, into L2
          for (int kb = 0; kb < kF / 64; ++kb)
            for (int z = 0; z < 2; ++z) tma_prefetch_3d(&tm_wb, h0 + kPrefetch * kHC, kb * 64, z);
        for (int kb = 0; kb < kF / 64; ++kb, ++it) {
          const int st = it % kB1Stages;
          mbar_wait(&b1empty[st], ((uint32_t)(it / kB1Stages) & 1u) ^ 1u);
          mbar_expect_tx(&b1full[st], kB1Stage);
          uint8_t* dst = sB1 + st * kB1Stage;
          tma_load_3d(dst, &tm_wb, &b1full[st], h0, kb * 64, 0);
          tma_load_3d(dst + kHC * 128, &tm_wb, &b1full[st], h0, kb * 64, 1);
        }
      }
    }
  } else if (warp == 2 + kEW) {
    if (lane == 0) {
      // ---------------- out-projection weight producer
      for (int c = 0; c < nc; ++c) {
        const int h0 = h_begin + c * kHC;
        if (c + 1 < nc)
          for (int j = 0; j < kF / 64; ++j) tma_prefetch_3d(&tm_wo, j * 64, h0 + kHC, 0);
        // in n-halves: half 0 of chunk c refills while MMA2(c-1) still works on
        // half 1 (a single 32 KB buffer put the weight load between every two
        // chunks' MMA2s)
        for (int q = 0; q < 2; ++q) {
          mbar_wait(&b2empty[q], ((uint32_t)c & 1u) ^ 1u);
          mbar_expect_tx(&b2full[q], kB2Bytes / 2);
          for (int j = 2 * q; j < 2 * q + 2; ++j)
            tma_load_3d(sB2 + j * 8192, &tm_wo, &b2full[q], j * 64, h0, 0);
        }
      }
    }
  } else if (warp == 3 + kEW) {
    if (lane == 0) {
      // ---------------- store warp: ff and D_z of each chunk to global once the
      // epilogue warps have staged them; frees the staging tiles for the next
      // chunk once the copies have read them
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_ff) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_d) : "memory");
      for (int c = 0; c < nc; ++c) {
        const int h0 = h_begin + c * kHC;
        mbar_wait(staged, (uint32_t)c & 1u);
        tma_store_3d(&tm_ff, sA2, h0, m0, 0);
        tma_store_3d(&tm_d, sD, h0, m0, 0);
        tma_store_3d(&tm_d, sD + kBM * 128, h0, m0, 1);
        bulk_commit();
        bulk_wait_read<0>();
        mbar_arrive(sfree);
      }
      bulk_wait_all();
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer
      // MMA1 computes both branches in one N = 128 instruction: the two 64-wide
      // branch boxes of a stage sit 8 KB apart, i.e. two MN atoms (LBO 8192),
      // landing in acc1 columns [0, 64) and [64, 128).  Descriptors are
      // built once; the per-step offsets go into the 14-bit address field.
      constexpr uint32_t id1 = idesc_f16(kBM, 2 * kHC, 0, 1);
      constexpr uint32_t id2 = idesc_f16(kBM, kF, 0, 1);
      const uint64_t d_a1 = sdesc(smem_u32(sA1), 16, 1024, kLayoutSW128);
      const uint64_t d_b1 = sdesc(smem_u32(sB1), 8192, 1024, kLayoutSW128);
      const uint64_t d_a2 = sdesc(smem_u32(sA2), 16, 1024, kLayoutSW128);
      const uint64_t d_b2 = sdesc(smem_u32(sB2), 8192, 1024, kLayoutSW128);
      mbar_wait(a1full, 0);
      tc_fence_after();
      int it = 0;
      for (int c = 0; c < nc; ++c) {  // MMA1(c), as soon as acc1[c & 1] is free
        const int b = c & 1;
        mbar_wait(&tempty1[b], ((uint32_t)(c >> 1) & 1u) ^ 1u);
        tc_fence_after();
        for (int kb = 0; kb < kF / 64; ++kb, ++it) {
          const int st = it % kB1Stages;
          mbar_wait(&b1full[st], (uint32_t)(it / kB1Stages) & 1u);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            tc_mma_f16(tmem + (uint32_t)(b * 2 * kHC),
                       d_a1 + (uint64_t)((kb * 16384 + kk * 32) >> 4),
                       d_b1 + (uint64_t)((st * kB1Stage + kk * 2048) >> 4), id1,
                       (kb > 0 || kk > 0) ? 1u : 0u);
          tc_commit(&b1empty[st]);
        }
        tc_commit(&tfull1[b]);
      }
      (void)id2;
      (void)d_a2;
      (void)d_b2;
    }
  } else if (warp == 4 + kEW) {
    if (lane == 0) {
      // ---------------- MMA2 issuer (its own thread: MMA1 never waits behind
      // an epilogue hand-off; the two write disjoint TMEM accumulators)
      // two N = 128 halves per chunk (columns 0-127, 128-255 of acc2): every
      // output column still accumulates the same 16-deep steps in the same order
      constexpr uint32_t id2 = idesc_f16(kBM, kF / 2, 0, 1);
      const uint64_t d_a2 = sdesc(smem_u32(sA2), 16, 1024, kLayoutSW128);
      const uint64_t d_b2 = sdesc(smem_u32(sB2), 8192, 1024, kLayoutSW128);
      for (int p = 0; p < nc; ++p) {  // acc2 += ff(p) . W_out[chunk p]
        mbar_wait(staged, (uint32_t)p & 1u);
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          mbar_wait(&b2full[q], (uint32_t)p & 1u);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            tc_mma_f16(tmem + 256u + (uint32_t)(q * kF / 2), d_a2 + (uint64_t)((kk * 32) >> 4),
                       d_b2 + (uint64_t)((q * 16384 + kk * 2048) >> 4), id2,
                       (p > 0 || kk > 0) ? 1u : 0u);
          tc_commit(&b2empty[q]);
        }
        tc_commit(a2empty);
      }
      tc_commit(t2full);
    }
  } else if (warp < 2 + kEW) {
    // ---------------- epilogue (TMEM lane quadrant = warp % 4)
    const int quad = warp & 3;
    const int half = (warp - 2) >> 2;  // columns half*kCW .. +kCW of each chunk
    const int r = quad * 32 + lane;    // tile row
    const uint32_t tq = tmem + ((uint32_t)(quad * 32) << 16);
    // the slice's branch biases, staged once in shared memory (global loads
    // right behind the TMEM loads exposed their L2 latency every chunk)
    for (int e = threadIdx.x - 64; e < 2 * hs; e += 32 * kEW)
      sBiasT[e] = b0[(e >= hs ? sBias : 0) + h_begin + (e >= hs ? e - hs : e)];
    named_bar(2, 32 * kEW);
    for (int c = 0; c < nc; ++c) {
      const int b = c & 1;
      const int h0 = h_begin + c * kHC;
      float4 bc0[kCW / 4], bc1[kCW / 4];
      {  // LDS.128 through the shared window (generic loads cost 64-bit address math)
        const uint32_t q0 = smem_u32(sBiasT + c * kHC + half * kCW);
        const uint32_t q1 = smem_u32(sBiasT + hs + c * kHC + half * kCW);
#pragma unroll
        for (int j = 0; j < kCW / 4; ++j) {
          asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                       : "=f"(bc0[j].x), "=f"(bc0[j].y), "=f"(bc0[j].z), "=f"(bc0[j].w)
                       : "r"(q0 + 16u * j));
          asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                       : "=f"(bc1[j].x), "=f"(bc1[j].y), "=f"(bc1[j].z), "=f"(bc1[j].w)
                       : "r"(q1 + 16u * j));
        }
      }
      mbar_wait(&tfull1[b], (uint32_t)(c >> 1) & 1u);
      tc_fence_after();
      float v0[kCW], v1[kCW];
      tmem_ldn<kCW>(tq + (uint32_t)(b * 2 * kHC + half * kCW), v0);
      tmem_ldn<kCW>(tq + (uint32_t)(b * 2 * kHC + kHC + half * kCW), v1);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty1[b]);  // acc1[b] may take chunk c+2
      // EpiBranchActH's arithmetic, in its order
#pragma unroll
      for (int j = 0; j < kCW / 4; ++j) {
        const float4 a = bc0[j], bq = bc1[j];
        v0[4 * j] = v0[4 * j] + a.x; v0[4 * j + 1] = v0[4 * j + 1] + a.y;
        v0[4 * j + 2] = v0[4 * j + 2] + a.z; v0[4 * j + 3] = v0[4 * j + 3] + a.w;
        v1[4 * j] = v1[4 * j] + bq.x; v1[4 * j + 1] = v1[4 * j + 1] + bq.y;
        v1[4 * j + 2] = v1[4 * j + 2] + bq.z; v1[4 * j + 3] = v1[4 * j + 3] + bq.w;
      }
      float f[kCW], p[kCW];
#pragma unroll
      for (int j = 0; j < kCW; ++j) {
        p[j] = v0[j] * v1[j];
        gelu_pair(p[j], f[j], p[j]);
      }
      // staging free: MMA2(c-1) done reading ff, the TMA stores of c-1 done
      // reading ff / D
      mbar_wait(a2empty, ((uint32_t)c & 1u) ^ 1u);
      mbar_wait(sfree, ((uint32_t)c & 1u) ^ 1u);
      put_row_h_sw128<kCW>(sA2, r, half * kCW / 8, f);
#pragma unroll
      for (int j = 0; j < kCW; ++j) f[j] = p[j] * v1[j];  // D_0 = GeLU' * H_1
      put_row_h_sw128<kCW>(sD, r, half * kCW / 8, f);
#pragma unroll
      for (int j = 0; j < kCW; ++j) f[j] = p[j] * v0[j];  // D_1 = GeLU' * H_0
      put_row_h_sw128<kCW>(sD + kBM * 128, r, half * kCW / 8, f);
      fence_async_smem();  // generic-proxy writes -> the MMA / TMA (async proxy)
      __syncwarp();
      if (lane == 0) mbar_arrive(staged);
    }
    // acc2 (this slice's out-projection partial) -> own shared memory, fp32
    // rows padded to kF + 4 floats (conflict-free row-per-thread writes);
    // every operand buffer is dead by now (t2full: all MMAs done)
    mbar_wait(t2full, 0);
    tc_fence_after();
  }
  tc_fence_before();
  __syncthreads();  // the store warp has drained its TMA stores, every MMA is done
  constexpr int kLd = kF + 4;
  float* sP = reinterpret_cast<float*>(smem);
  if (warp >= 2 && warp < 2 + kEW) {
    const int quad = warp & 3, half = (warp - 2) >> 2, r = quad * 32 + lane;
    const uint32_t tq = tmem + ((uint32_t)(quad * 32) << 16);
#pragma unroll 1
    for (int cb = half * (kF * 4 / kEW); cb < (half + 1) * (kF * 4 / kEW); cb += 32) {
      float v[32];
      tmem_ld32(tq + 256u + (uint32_t)cb, v);
      const uint32_t dst = smem_u32(sP + r * kLd + cb);
#pragma unroll
      for (int j = 0; j < 8; ++j)
        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(dst + 16 * j), "f"(v[4 * j]),
                     "f"(v[4 * j + 1]), "f"(v[4 * j + 2]), "f"(v[4 * j + 3])
                     : "memory");
    }
  }
  cluster_sync_all();
  // the kFusedSplit CTAs of this row tile form the cluster; CTA q sums column
  // quarter q of the four partials in rank order -- ((p0 + p1) + p2) + p3,
  // then + bias, then + residual: k_splitk_reduce's order, bit for bit -- and
  // writes the block output (tf32-rounded when it feeds a tf32 GEMM)
  {
    const uint32_t q = cluster_rank();
    constexpr int kQ = kF / kFusedSplit;       // 64 columns
    for (int e = threadIdx.x; e < kBM * kQ / 4; e += kThreads) {
      const int row = e / (kQ / 4), col = (int)q * kQ + 4 * (e % (kQ / 4));
      const int m = m0 + row;
      const uint32_t la = smem_u32(sP + row * kLd + col);
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int rk = 0; rk < kFusedSplit; ++rk) {
        uint32_t ra;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(rk));
        float4 w;
        asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(w.x), "=f"(w.y), "=f"(w.z), "=f"(w.w)
                     : "r"(ra)
                     : "memory");
        if (rk == 0) {
          a = w;
        } else {
          a.x += w.x; a.y += w.y; a.z += w.z; a.w += w.w;
        }
      }
      if (m < Bl) {
        const float4 b = *reinterpret_cast<const float4*>(bias_out + col);
        const float4 x = *reinterpret_cast<const float4*>(resid + (int64_t)m * kF + col);
        a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
        a.x += x.x; a.y += x.y; a.z += x.z; a.w += x.w;
        if (rt) {
          a.x = tf32_rna(a.x); a.y = tf32_rna(a.y); a.z = tf32_rna(a.z); a.w = tf32_rna(a.w);
        }
        *reinterpret_cast<float4*>(out + (int64_t)m * kF + col) = a;
      }
    }
  }
  cluster_sync_all();  // no CTA leaves while a peer may still read its partial
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// fp16 [c2][rows][inner] store map, box {64, 128, 1}, 128B swizzle (the
// K-major MMA operand layout of one 64-wide chunk)
inline bool make_store_map_h64(CUtensorMap* map, const void* base, uint64_t inner, uint64_t rows,
                               uint64_t batch) {
  cuuint64_t dims[3] = {inner, rows, batch};
  cuuint64_t strides[2] = {inner * 2, inner * rows * 2};
  cuuint32_t box[3] = {64, 128, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  PfnEncodeTiled enc = encode_tiled_fn();
  return enc && enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, (void*)base, dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
                    CUDA_SUCCESS;
}

struct FusedMapCache {
  std::mutex mu;
  std::map<std::tuple<const void*, uint64_t, uint64_t, uint64_t>, CUtensorMap> maps;
  bool get(CUtensorMap* out, const void* base, uint64_t inner, uint64_t rows, uint64_t batch) {
    auto key = std::make_tuple(base, inner, rows, batch);
    std::lock_guard<std::mutex> g(mu);
    auto it = maps.find(key);
    if (it == maps.end()) {
      CUtensorMap m{};
      if (!make_store_map_h64(&m, base, inner, rows, batch)) return false;
      it = maps.emplace(key, m).first;
    }
    *out = it->second;
    return true;
  }
};

inline FusedMapCache& fused_map_cache() {
  static FusedMapCache c;
  return c;
}

// shapes the fused kernel covers (else the caller takes the unfused path)
inline bool mbrb_fused_ok(int F, int H, int K) {
  return K == 2 && F == mf::kF && H % (kFusedSplit * mf::kHC) == 0 &&
         H / kFusedSplit <= mf::kMaxSlice;
}

// x0h [Bl][F] fp16, Wb = branch-0 weight [F][H] fp16 (branch 1 at + sW),
// Wo [H][F] fp16, b0 fp32 bias of branch 0 (branch 1 at + sW); writes ff
// [Bl][H], D [2][Bl][H] (fp16) and out [Bl][F] = ff . Wo + bias_out + resid
// (rounded to tf32 when rt).  Clusters of kFusedSplit CTAs (the H slices of
// one row tile) reduce the slices over DSMEM.
inline int mbrb_fwd_fused(const __half* x0h, const __half* Wb, int64_t sW, const __half* Wo,
                          const float* b0, int Bl, int H, __half* ff, __half* D,
                          const float* bias_out, const float* resid, float* out, int rt,
                          cudaStream_t st) {
  using namespace mf;
  CUtensorMap tx, tw, to, tf, td;
  int r = tmap_cache().get(&tx, x0h, kF, (uint64_t)Bl, 1, kF, 0, 64, kBM, 2);
  if (r == EDPC_OK) r = tmap_cache().get(&tw, Wb, (uint64_t)H, kF, 2, (uint64_t)H, (uint64_t)sW, 64, 64, 3);
  if (r == EDPC_OK) r = tmap_cache().get(&to, Wo, kF, (uint64_t)H, 1, kF, 0, 64, 64, 3);
  if (r != EDPC_OK) return r;
  if (!fused_map_cache().get(&tf, ff, (uint64_t)H, (uint64_t)Bl, 1) ||
      !fused_map_cache().get(&td, D, (uint64_t)H, (uint64_t)Bl, 2)) {
    set_error("mbrb_fwd_fused: fp16 store maps not encodable");
    return EDPC_ERR_CUDA;
  }
  static bool attr[16] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr[dev & 15]) {
    cudaFuncSetAttribute(k_mbrb_fwd_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    attr[dev & 15] = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(cdiv(Bl, kBM) * kFusedSplit));
  cfg.blockDim = dim3((unsigned)kThreads);
  cfg.dynamicSmemBytes = (size_t)kSmemBytes;
  cfg.stream = st;
  cudaLaunchAttribute attr2[2];
  attr2[0].id = cudaLaunchAttributeClusterDimension;
  attr2[0].val.clusterDim.x = (unsigned)kFusedSplit;
  attr2[0].val.clusterDim.y = 1;
  attr2[0].val.clusterDim.z = 1;
  attr2[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr2[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr2;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_mbrb_fwd_fused, tx, tw, to, tf, td, b0, sW, Bl, H,
                                     bias_out, resid, out, rt);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("k_mbrb_fwd_fused launch: ") + cudaGetErrorString(e));
    return EDPC_ERR_CUDA;
  }
  return EDPC_OK;
}



// ===================================================================
// Fused MBRB backward (model.py:105-121): the out-projection dgrad, the
// product-rule epilogue and the branch dgrad in one kernel.
//
//   g_ff  = g_up . W_out^T                      (g_up fp16 [Bl][F], per H chunk)
//   g_H_z = g_ff * D_z                          (D_z from the forward; stored fp16:
//                                                the branch weight gradients)
//   g_x0  = sum_z g_H_z . W_z^T                 (accumulated over the CTA's H slice)
//
// Same skeleton as the forward: a CTA owns a 128-row tile and one H slice in
// chunks of 64; MMA1 (N = 64, K = F) into a double-buffered TMEM accumulator,
// the epilogue multiplies by the D_z tiles that a loader warp TMA-loads into
// double-buffered staging tiles and writes g_H_z back in place -- the staging
// tiles then serve as the A operands of MMA2 (acc2 += g_H_z . W_z^T, N = F)
// and as the source of the g_H_z TMA stores.  The 4 slices of a row tile are
// a cluster and reduce over DSMEM in rank order.  MMA2 walks each 64-deep
// block as branch 0 then branch 1, the order of the unfused split-K dgrad
// (tc_gemm.cuh kBatchSum), so the result is bit-identical to it.
namespace mb {
constexpr int kBM = 128, kF = 256, kHC = 64, kEW = 16, kCW = kHC / (kEW / 4);
constexpr int kB1Stages = 4;
constexpr int kThreads = 32 * (2 + kEW + 3);  // + W_z producer, store/D loader, MMA2 issuer
constexpr int kA1Bytes = kBM * kF * 2;        // g_up tile, 64 KB
constexpr int kB1Stage = kHC * 64 * 2;        // W_out rows of the chunk, one 64-deep k-block: 8 KB
constexpr int kB2Bytes = 2 * kF * kHC * 2;    // both branches' W_z^T blocks: 64 KB
constexpr int kTile = kBM * kHC * 2;          // one 128 x 64 fp16 tile: 16 KB
constexpr int kOffA1 = 0;
constexpr int kOffB1 = kOffA1 + kA1Bytes;
constexpr int kOffB2 = kOffB1 + kB1Stages * kB1Stage;
constexpr int kOffS = kOffB2 + kB2Bytes;      // staging [2 buffers][2 branches] tiles
constexpr int kOffBar = kOffS + 4 * kTile;
constexpr int kSmemBytes = 1024 + kOffBar + 256;
}  // namespace mb

__global__ void __launch_bounds__(mb::kThreads, 1)
k_mbrb_bwd_fused(const __grid_constant__ CUtensorMap tm_g, const __grid_constant__ CUtensorMap tm_wo,
                 const __grid_constant__ CUtensorMap tm_wb, const __grid_constant__ CUtensorMap tm_d,
                 const __grid_constant__ CUtensorMap tm_gh, int Bl, int H, float* __restrict__ out) {
  using namespace mb;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA1 = smem + kOffA1;
  uint8_t* sB1 = smem + kOffB1;
  uint8_t* sB2 = smem + kOffB2;
  uint8_t* sS = smem + kOffS;  // buffer u, branch z at sS + (2u + z) * kTile
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + kOffBar);
  uint64_t* a1full = bar;
  uint64_t* b1full = bar + 1;
  uint64_t* b1empty = b1full + kB1Stages;
  uint64_t* b2full = b1empty + kB1Stages;  // [2] W_0^T / W_1^T blocks of a chunk
  uint64_t* b2empty = b2full + 2;          // [2]
  uint64_t* tfull1 = b2empty + 2;  // [2]
  uint64_t* tempty1 = tfull1 + 2;  // [2]
  uint64_t* dfull = tempty1 + 2;   // [2] D tiles of a chunk loaded into staging buffer u
  uint64_t* staged = dfull + 2;    // g_H of a chunk written (one arrive per epilogue warp)
  uint64_t* a2empty = staged + 1;  // MMA2 done with a chunk's staging buffer
  uint64_t* sdone = a2empty + 1;   // the store warp has finished a chunk (all its waits for it)
  uint64_t* t2full = sdone + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(t2full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x / kFusedSplit, split = blockIdx.x % kFusedSplit;
  const int m0 = tile * kBM;
  const int hs = H / kFusedSplit;
  const int h_begin = split * hs;
  const int nc = hs / kHC;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_g) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_wo) : "memory");
    mbar_init(a1full, 1);
    for (int s = 0; s < kB1Stages; ++s) {
      mbar_init(&b1full[s], 1);
      mbar_init(&b1empty[s], 1);
    }
    for (int q = 0; q < 2; ++q) {
      mbar_init(&b2full[q], 1);
      mbar_init(&b2empty[q], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull1[b], 1);
      mbar_init(&tempty1[b], kEW);
      mbar_init(&dfull[b], 1);
    }
    mbar_init(staged, kEW);
    mbar_init(a2empty, 1);
    mbar_init(sdone, 1);
    mbar_init(t2full, 1);
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
  if (warp == 0 && lane == 0) {  // weights into L2 while the predecessor drains
    for (int c = 0; c < 2 && c < nc; ++c) {
      for (int kb = 0; kb < kF / 64; ++kb) tma_prefetch_3d(&tm_wo, kb * 64, h_begin + c * kHC, 0);
      for (int z = 0; z < 2; ++z) tma_prefetch_3d(&tm_wb, h_begin + c * kHC, 0, z);
    }
  }
  pdl_entry();

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- producer: g_up tile once, W_out rows per chunk
      mbar_expect_tx(a1full, kA1Bytes);
#pragma unroll
      for (int kb = 0; kb < kF / 64; ++kb) tma_load_3d(sA1 + kb * 16384, &tm_g, a1full, kb * 64, m0, 0);
      int it = 0;
      for (int c = 0; c < nc; ++c) {
        const int h0 = h_begin + c * kHC;
        if (c + 2 < nc)
          for (int kb = 0; kb < kF / 64; ++kb) tma_prefetch_3d(&tm_wo, kb * 64, h0 + 2 * kHC, 0);
        for (int kb = 0; kb < kF / 64; ++kb, ++it) {
          const int st = it % kB1Stages;
          mbar_wait(&b1empty[st], ((uint32_t)(it / kB1Stages) & 1u) ^ 1u);
          mbar_expect_tx(&b1full[st], kB1Stage);
          tma_load_3d(sB1 + st * kB1Stage, &tm_wo, &b1full[st], kb * 64, h0, 0);
        }
      }
    }
  } else if (warp == 2 + kEW) {
    if (lane == 0) {
      // ---------------- W_z^T producer (both branches, K-major boxes of 64 x 256)
      for (int c = 0; c < nc; ++c) {
        const int h0 = h_begin + c * kHC;
        if (c + 1 < nc)
          for (int z = 0; z < 2; ++z) tma_prefetch_3d(&tm_wb, h0 + kHC, 0, z);
        // per branch: W_0^T of chunk c refills while MMA2(c-1) still works on
        // branch 1 (one 64 KB buffer put the load between every two chunks)
        for (int z = 0; z < 2; ++z) {
          mbar_wait(&b2empty[z], ((uint32_t)c & 1u) ^ 1u);
          mbar_expect_tx(&b2full[z], kB2Bytes / 2);
          tma_load_3d(sB2 + z * (kF * 128), &tm_wb, &b2full[z], h0, 0, z);
        }
      }
    }
  } else if (warp == 3 + kEW) {
    if (lane == 0) {
      // ---------------- D loader + g_H store warp
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_d) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_gh) : "memory");
      auto load_d = [&](int c) {
        const int u = c & 1;
        mbar_expect_tx(&dfull[u], 2 * kTile);
        for (int z = 0; z < 2; ++z)
          tma_load_3d(sS + (2 * u + z) * kTile, &tm_d, &dfull[u], h_begin + c * kHC, m0, z);
      };
      for (int c = 0; c < 2 && c < nc; ++c) load_d(c);
      for (int c = 0; c < nc; ++c) {
        const int u = c & 1, h0 = h_begin + c * kHC;
        mbar_wait(staged, (uint32_t)c & 1u);
        for (int z = 0; z < 2; ++z) tma_store_3d(&tm_gh, sS + (2 * u + z) * kTile, h0, m0, z);
        bulk_commit();
        if (c + 2 < nc) {  // buffer u takes chunk c+2 once the stores and MMA2(c) have read it
          bulk_wait_read<0>();
          mbar_wait(a2empty, (uint32_t)c & 1u);
          load_d(c + 2);
        }
        mbar_arrive(sdone);  // iteration c done: both of its parity waits are behind it
      }
      bulk_wait_all();
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA1 issuer: g_ff(c) = g_up . W_out[chunk c]^T
      constexpr uint32_t id1 = idesc_f16(kBM, kHC, 0, 0);
      const uint64_t d_a1 = sdesc(smem_u32(sA1), 16, 1024, kLayoutSW128);
      const uint64_t d_b1 = sdesc(smem_u32(sB1), 16, 1024, kLayoutSW128);
      mbar_wait(a1full, 0);
      tc_fence_after();
      int it = 0;
      for (int c = 0; c < nc; ++c) {
        const int b = c & 1;
        mbar_wait(&tempty1[b], ((uint32_t)(c >> 1) & 1u) ^ 1u);
        tc_fence_after();
        for (int kb = 0; kb < kF / 64; ++kb, ++it) {
          const int st = it % kB1Stages;
          mbar_wait(&b1full[st], (uint32_t)(it / kB1Stages) & 1u);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            tc_mma_f16(tmem + (uint32_t)(b * kHC), d_a1 + (uint64_t)((kb * 16384 + kk * 32) >> 4),
                       d_b1 + (uint64_t)((st * kB1Stage + kk * 32) >> 4), id1,
                       (kb > 0 || kk > 0) ? 1u : 0u);
          tc_commit(&b1empty[st]);
        }
        tc_commit(&tfull1[b]);
      }
    }
  } else if (warp == 4 + kEW) {
    if (lane == 0) {
      // ---------------- MMA2 issuer: acc2 += g_H_0 . W_0^T + g_H_1 . W_1^T per chunk
      constexpr uint32_t id2 = idesc_f16(kBM, kF, 0, 0);
      const uint64_t d_s = sdesc(smem_u32(sS), 16, 1024, kLayoutSW128);
      const uint64_t d_b2 = sdesc(smem_u32(sB2), 16, 1024, kLayoutSW128);
      for (int c = 0; c < nc; ++c) {
        const int u = c & 1;
        mbar_wait(staged, (uint32_t)c & 1u);
#pragma unroll
        for (int z = 0; z < 2; ++z) {
          mbar_wait(&b2full[z], (uint32_t)c & 1u);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            tc_mma_f16(tmem + 256u, d_s + (uint64_t)(((2 * u + z) * kTile + kk * 32) >> 4),
                       d_b2 + (uint64_t)((z * (kF * 128) + kk * 32) >> 4), id2,
                       (c > 0 || z > 0 || kk > 0) ? 1u : 0u);
          tc_commit(&b2empty[z]);
        }
        tc_commit(a2empty);
      }
      tc_commit(t2full);
    }
  } else if (warp < 2 + kEW) {
    // ---------------- epilogue: g_H_z = g_ff * D_z, in place in the staging tiles
    const int quad = warp & 3, half = (warp - 2) >> 2, r = quad * 32 + lane;
    const uint32_t tq = tmem + ((uint32_t)(quad * 32) << 16);
    for (int c = 0; c < nc; ++c) {
      const int b = c & 1, u = c & 1;
      mbar_wait(&tfull1[b], (uint32_t)(c >> 1) & 1u);
      tc_fence_after();
      float g[kCW];
      tmem_ldn<kCW>(tq + (uint32_t)(b * kHC + half * kCW), g);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty1[b]);
      mbar_wait(&dfull[u], (uint32_t)(c >> 1) & 1u);
#pragma unroll
      for (int z = 0; z < 2; ++z) {
        const uint32_t row = smem_u32(sS + (2 * u + z) * kTile) + (uint32_t)(r * 128);
#pragma unroll
        for (int jj = 0; jj < kCW / 8; ++jj) {
          const uint32_t a = row + (uint32_t)(((half * kCW / 8 + jj) ^ (r & 7)) << 4);
          uint32_t w[4];
          asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3])
                       : "r"(a));
#pragma unroll
          for (int q = 0; q < 4; ++q) {  // EpiBwdActH: g_H = g_ff * D, rounded to fp16
            const float2 d = __half22float2(*reinterpret_cast<const __half2*>(&w[q]));
            __half2 o = __floats2half2_rn(g[8 * jj + 2 * q] * d.x, g[8 * jj + 2 * q + 1] * d.y);
            w[q] = *reinterpret_cast<uint32_t*>(&o);
          }
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(w[0]), "r"(w[1]),
                       "r"(w[2]), "r"(w[3])
                       : "memory");
        }
      }
      fence_async_smem();
      // Parity waits alias when a barrier completes two phases before its
      // waiter looks: chunk c's `staged` arrivals wait until MMA2(c-1) has
      // completed (the MMA2 issuer is past staged(c-1)) and the store warp has
      // finished iteration c-1 (past its staged(c-1) and a2empty(c-1) waits),
      // so neither `staged` nor `a2empty` can lap the thread waiting on it.
      // (Without this the epilogue, which needs neither of them to proceed,
      // could run two chunks ahead and deadlock the CTA.)
      if (c > 0) {
        mbar_wait(a2empty, (uint32_t)(c - 1) & 1u);
        mbar_wait(sdone, (uint32_t)(c - 1) & 1u);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(staged);
    }
    mbar_wait(t2full, 0);
    tc_fence_after();
  }
  tc_fence_before();
  __syncthreads();
  constexpr int kLd = kF + 4;
  float* sP = reinterpret_cast<float*>(smem);
  if (warp >= 2 && warp < 2 + kEW) {
    const int quad = warp & 3, half = (warp - 2) >> 2, r = quad * 32 + lane;
    const uint32_t tq = tmem + ((uint32_t)(quad * 32) << 16);
#pragma unroll 1
    for (int cb = half * (kF * 4 / kEW); cb < (half + 1) * (kF * 4 / kEW); cb += 32) {
      float v[32];
      tmem_ld32(tq + 256u + (uint32_t)cb, v);
      const uint32_t dst = smem_u32(sP + r * kLd + cb);
#pragma unroll
      for (int j = 0; j < 8; ++j)
        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(dst + 16 * j), "f"(v[4 * j]),
                     "f"(v[4 * j + 1]), "f"(v[4 * j + 2]), "f"(v[4 * j + 3])
                     : "memory");
    }
  }
  cluster_sync_all();
  {  // column quarter q of the 4 slice partials, in rank order (k_splitk_reduce's)
    const uint32_t q = cluster_rank();
    constexpr int kQ = kF / kFusedSplit;
    for (int e = threadIdx.x; e < kBM * kQ / 4; e += kThreads) {
      const int row = e / (kQ / 4), col = (int)q * kQ + 4 * (e % (kQ / 4));
      const int m = m0 + row;
      const uint32_t la = smem_u32(sP + row * kLd + col);
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int rk = 0; rk < kFusedSplit; ++rk) {
        uint32_t ra;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(rk));
        float4 w;
        asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(w.x), "=f"(w.y), "=f"(w.z), "=f"(w.w)
                     : "r"(ra)
                     : "memory");
        if (rk == 0) {
          a = w;
        } else {
          a.x += w.x; a.y += w.y; a.z += w.z; a.w += w.w;
        }
      }
      if (m < Bl) *reinterpret_cast<float4*>(out + (int64_t)m * kF + col) = a;
    }
  }
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// guph [Bl][F] fp16 (the block-output gradient), Wo [H][F] fp16, Wb = branch-0
// weight [F][H] fp16 (branch 1 at + sW), D [2][Bl][H] fp16 from the forward;
// writes g_H [2][Bl][H] fp16 and out [Bl][F] fp32 = sum_z g_H_z . W_z^T.
inline int mbrb_bwd_fused(const __half* guph, const __half* Wo, const __half* Wb, int64_t sW,
                          const __half* D, __half* GH, int Bl, int H, float* out, cudaStream_t st) {
  using namespace mb;
  CUtensorMap tg, to, tw, td, th;
  int r = tmap_cache().get(&tg, guph, kF, (uint64_t)Bl, 1, kF, 0, 64, kBM, 2);
  if (r == EDPC_OK) r = tmap_cache().get(&to, Wo, kF, (uint64_t)H, 1, kF, 0, 64, 64, 2);
  if (r == EDPC_OK) r = tmap_cache().get(&tw, Wb, (uint64_t)H, kF, 2, (uint64_t)H, (uint64_t)sW, 64, 256, 2);
  if (r != EDPC_OK) return r;
  if (!fused_map_cache().get(&td, D, (uint64_t)H, (uint64_t)Bl, 2) ||
      !fused_map_cache().get(&th, GH, (uint64_t)H, (uint64_t)Bl, 2)) {
    set_error("mbrb_bwd_fused: fp16 tile maps not encodable");
    return EDPC_ERR_CUDA;
  }
  static bool attr[16] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr[dev & 15]) {
    cudaFuncSetAttribute(k_mbrb_bwd_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    attr[dev & 15] = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(cdiv(Bl, kBM) * kFusedSplit));
  cfg.blockDim = dim3((unsigned)kThreads);
  cfg.dynamicSmemBytes = (size_t)kSmemBytes;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)kFusedSplit;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_mbrb_bwd_fused, tg, to, tw, td, th, Bl, H, out);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("k_mbrb_bwd_fused launch: ") + cudaGetErrorString(e));
    return EDPC_ERR_CUDA;
  }
  return EDPC_OK;
}

}  // namespace edpc
