// tcgen05 / TMA / TMEM GEMM for sm_100a -- the fast path of every per-step
// contraction of the EDPC predictor and its online update.
//
//   D[M x N] (fp32, TMEM) = sum_k A[M x K] * B[K x N], kind::tf32 (fp32 in HBM)
//
// One CTA per 128 x BN output tile, warp-specialised:
//   warp 0      TMA producer: 128B-swizzled tiles of A and B into a
//               kStages-deep shared-memory ring (mbarrier full/empty pairs)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer (4 MMAs of
//               K=8 per 32-wide K block); tcgen05.commit frees ring slots
//   warps 2..9  epilogue (two warps per TMEM lane quadrant, alternating
//               32-column chunks): tcgen05.ld 32x32b.x32 -> registers -> fused
//               epilogue functor (bias, residual, GeLU/product-rule backward,
//               lane-group weight-gradient partials) -> global
// Operands may be K-major or MN-major (the instruction descriptor's
// transpose bits), so activations stored [lanes][features] serve directly as
// the MN-major operands of the weight-gradient GEMMs (K = lanes).
// The MMA order over K is fixed, so results are bitwise reproducible.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <type_traits>

#include "common.cuh"
#include "tc_types.cuh"

namespace edpc {

inline bool tc_compiled() { return true; }
inline bool tc_enabled_env() {
  const char* e = getenv("EDPC_TCGEN05");
  return !(e && e[0] == '0');
}

constexpr int kTcBM = 128;
constexpr int kTcBK = 32;  // fp32 elements per 128-byte swizzle row
constexpr int kTcStages = 4;

// --------------------------------------------------------------- PTX helpers

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@p bra DONE_%=;\n\t"
      "bra WAIT_%=;\n\t"
      "DONE_%=:\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(0x989680)  // suspend-time hint: sleep, do not poll (ncu: spinning
      : "memory");                 // producer/MMA warps took ~10% of the issue slots)
}

// Polling wait (try_wait without a suspend-time hint: the thread re-polls
// instead of sleeping).  For waits on a tcgen05.commit arrival in latency-
// critical loops: a thread suspended with the hint was seen to resume late
// after such arrivals (the fused kernels' epilogues stalled on them).
__device__ __forceinline__ void mbar_wait_spin(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAITS_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@p bra DONES_%=;\n\t"
      "bra WAITS_%=;\n\t"
      "DONES_%=:\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// TMA bulk-tensor store of a 4D box from shared memory (bulk-group tracked)
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* map, const void* src, int c0, int c1,
                                             int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
          map),
      "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// the smem sources of all but the newest N committed groups may be reused
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// generic-proxy smem writes -> visible to the async (TMA) proxy
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// TMA load multicast to the CTAs of the cluster in cta_mask (same smem offset
// and mbarrier offset in every destination CTA)
__device__ __forceinline__ void tma_load_3d_mc(void* dst, const CUtensorMap* map, uint64_t* bar,
                                               int c0, int c1, int c2, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".multicast::cluster [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "h"(mask)
      : "memory");
}

__device__ __forceinline__ void tc_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"(mask)
      : "memory");
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}

// arrive on the mbarrier at the same offset in cluster CTA `rank`
__device__ __forceinline__ void mbar_arrive_cluster(uint64_t* bar, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"(rank));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote)
               : "memory");
}

__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tc_mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void tc_mma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                           uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// 32 lanes x 32 consecutive fp32 columns -> 32 registers per thread
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
}

// Shared-memory matrix descriptor (tcgen05 "version 1").
//   K-major : SWIZZLE_128B (layout 2): rows of 128 B (32 fp32 of K), 8-row
//             atoms 1024 B apart (SBO); K steps of 8 advance the start by 32 B
//   MN-major: tf32 admits only SWIZZLE_128B_BASE32B (layout 1): K-rows of
//             128 B (32 fp32 of M/N) swizzled in 32 B units over 4-row atoms
//             (SBO = 512 B), 32-wide MN blocks LBO apart; K steps of 8 rows
//             advance the start by 1024 B
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo,
                                          uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (Blackwell)
  d |= (uint64_t)layout << 61;
  return d;
}
constexpr uint32_t kLayoutSW128 = 2, kLayoutSW128Base32B = 1;

// instruction descriptor: D f32, A/B tf32 (format 2) or f16 (format 0),
// majors, N>>3, M>>4
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// fp16 operands (H): 128-byte smem rows hold 64 elements of K (K-major) or of
// M/N (MN-major, the standard SWIZZLE_128B layout: 64-wide MN atoms of 8
// K-rows, one TMA box of 64 x 64 per atom column); 4 MMAs of K = 16 per
// k-block, as the tf32 path's 4 of K = 8 -- same smem bytes per stage.
template <bool H>
__host__ __device__ constexpr int tc_bk() {
  return H ? 64 : 32;
}
constexpr uint32_t kMnH_LBO = 8192, kMnH_SBO = 1024;

// ------------------------------------------------------------------ shapes

// ------------------------------------------------------------------ kernel

// ZIN > 1: ZIN batches (the MBRB branches) are computed by the same CTA for
// the same (tm, tn) tile -- one A tile and ZIN B tiles per stage, ZIN
// accumulators per TMEM buffer -- so the epilogue sees all branches at once.
// Epilogue warps transpose each 32x32 accumulator block through shared
// memory (padded rows of 33) so that every global load/store of the
// epilogue is a coalesced 128-byte row segment.
// 32x32 transpose scratch, XOR-swizzled (element (r, c) at r*32 + (c ^ r)):
// conflict-free row writes and column reads without padding
constexpr int kTcTileFloats = 32 * 32;

// Epilogue functors that read extra inputs (residual, product-rule factors)
// set kTransposed and get the smem transpose; store-only epilogues keep the
// shared memory for one more pipeline stage.
template <class Epi, class = void>
struct EpiTransposed {
  static constexpr bool value = false;
};
template <class Epi>
struct EpiTransposed<Epi, std::void_t<decltype(Epi::kTransposed)>> {
  static constexpr bool value = Epi::kTransposed;
};

// TMA-store epilogues (Epi::kTmaStore).  Each epilogue warp owns kTsSlots
// 4 KB boxes of shared memory; a box holds one 32x32 block in the row-per-
// thread layout of tcgen05.ld (row = TMEM lane), 128B-swizzled, and leaves
// through a TMA bulk-tensor store.  ncu on the row-per-thread global stores
// showed the K=256 GEMMs bound by the LSU (each warp-wide STG.128 touches 32
// rows: ~256 L1 wavefronts per block, the store-free ablation ran 1.9x
// faster); a box costs 32 wavefronts of STS.128 and the copy engine writes
// whole lines.  Epilogues that read a second operand (kTsIn boxes per block,
// e.g. the stored GeLU' factors) get it TMA-loaded into slots 0..kTsIn-1
// before their tcgen05.ld and overwrite the slots in place.  The functor:
//   host:   bool store_maps(const TcShape&, TcStoreMap& c, TcStoreMap& d) const
//           (maps 0 and 1; false -> the kernel uses its non-TMA path)
//   device: template <class IO, int Z>
//           void ts_chunk(IO&, zb, zg, m, n0, float (&v)[Z][32]) const
//           void ts_in(i, zb, zg, int& c2, int& c3) const   (kTsIn > 0)
template <class Epi, class = void>
struct EpiTmaStore {
  static constexpr bool value = false;
};
template <class Epi>
struct EpiTmaStore<Epi, std::void_t<decltype(Epi::kTmaStore)>> {
  static constexpr bool value = Epi::kTmaStore;
};
template <class Epi, class = void>
struct EpiTsSlots {
  static constexpr int value = 1;
};
template <class Epi>
struct EpiTsSlots<Epi, std::void_t<decltype(Epi::kTsSlots)>> {
  static constexpr int value = Epi::kTsSlots;
};
template <class Epi, class = void>
struct EpiTsInBytes {
  static constexpr int value = 32 * 32 * 4;
};
template <class Epi>
struct EpiTsInBytes<Epi, std::void_t<decltype(Epi::kTsInBytes)>> {
  static constexpr int value = Epi::kTsInBytes;
};
template <class Epi, class = void>
struct EpiRequireTs {
  static constexpr bool value = false;
};
template <class Epi>
struct EpiRequireTs<Epi, std::void_t<decltype(Epi::kRequireTs)>> {
  static constexpr bool value = Epi::kRequireTs;
};
template <class Epi, class = void>
struct EpiTsIn {
  static constexpr int value = 0;
};
template <class Epi>
struct EpiTsIn<Epi, std::void_t<decltype(Epi::kTsIn)>> {
  static constexpr int value = Epi::kTsIn;
};
constexpr int kTsBoxBytes = 32 * 32 * 4;
// bytes per TMA-store slot: a 32x32 fp32 box by default; epilogues that only
// move fp16 boxes (2 KB) declare kTsSlotBytes = 2048 and get twice the slots
// -- twice the stores in flight -- in the same shared memory
template <class Epi, class = void>
struct EpiTsSlotBytes {
  static constexpr int value = kTsBoxBytes;
};
template <class Epi>
struct EpiTsSlotBytes<Epi, std::void_t<decltype(Epi::kTsSlotBytes)>> {
  static constexpr int value = Epi::kTsSlotBytes;
};
constexpr int kStagesMax = 4;

template <int BN, int ZIN = 1, bool TR = true, int EW = 8, int TSLOTS = 0, int TSB = kTsBoxBytes>
struct TcSmem {
  static constexpr int kABytes = kTcBM * kTcBK * 4;  // 16 KB
  static constexpr int kBBytes = BN * kTcBK * 4;
  static constexpr int kStageBytes = kABytes + ZIN * kBBytes;
  static constexpr int kTrBytes = TR ? EW * ZIN * kTcTileFloats * 4 : 0;
  static constexpr int kTsBytes = EW * TSLOTS * TSB;
  static constexpr int kEpiBytes = kTrBytes > kTsBytes ? kTrBytes : kTsBytes;
  static constexpr int kFixed = 1024 /*align*/ + 512 /*barriers*/ + kEpiBytes;
  static constexpr int kStages = (4 * kStageBytes + kFixed <= 232448)   ? 4
                                 : (3 * kStageBytes + kFixed <= 232448) ? 3
                                                                        : 2;
  static constexpr int kEpiOffset = kStages * kStageBytes;
  static constexpr int kBarOffset = kEpiOffset + kEpiBytes;
  static constexpr int kBytes = kStages * kStageBytes + kFixed;
  static constexpr int kCols = 2 * ZIN * BN;  // double-buffered accumulators
  static constexpr uint32_t kTmemCols =
      kCols <= 32 ? 32 : kCols <= 64 ? 64 : kCols <= 128 ? 128 : kCols <= 256 ? 256 : 512;
};

// Per-warp box writer of a TMA-store epilogue (see EpiTmaStore).
template <int NS, int SF = 1024>  // NS slots of SF floats
struct TsIo {
  float* slots;  // NS boxes of 32x32 floats
  const CUtensorMap* maps[2];
  int n0, m0;    // box origin (columns, rows)
  int* next;     // ring position (persists across blocks)
  int ib;        // first slot of this block's input boxes (in / put_at)
  // row `lane` of box `slot`: 16-byte chunk j at j ^ (lane & 7) (SWIZZLE_128B)
  // (32-bit shared-window addresses: STS/LDS, not generic 64-bit accesses)
  __device__ __forceinline__ void write_row(int slot, const float (&v)[32]) const {
    const int lane = threadIdx.x & 31;
    const uint32_t box = smem_u32(slots + slot * SF + lane * 32);
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(
                       box + (uint32_t)((j ^ (lane & 7)) << 4)),
                   "f"(v[4 * j]), "f"(v[4 * j + 1]), "f"(v[4 * j + 2]), "f"(v[4 * j + 3])
                   : "memory");
  }
  __device__ __forceinline__ void in(int slot, float (&v)[32]) const {
    const int lane = threadIdx.x & 31;
    const uint32_t box = smem_u32(slots + (ib + slot) * SF + lane * 32);
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                   : "=f"(v[4 * j]), "=f"(v[4 * j + 1]), "=f"(v[4 * j + 2]), "=f"(v[4 * j + 3])
                   : "r"(box + (uint32_t)((j ^ (lane & 7)) << 4))
                   : "memory");
  }
  __device__ __forceinline__ void issue(int slot, int map, int c2, int c3) const {
    fence_async_smem();
    __syncwarp();
    if ((threadIdx.x & 31) == 0) {
      tma_store_4d(maps[map], slots + slot * SF, n0, m0, c2, c3);  // rows past M are clipped
      bulk_commit();
    }
  }
  // fp16 boxes: rows of 64 B (32 halves), SWIZZLE_64B: 16-byte chunk j of
  // row r at j ^ ((r >> 1) & 3) -- conflict-free for 8 rows per phase
  __device__ __forceinline__ void write_row_h(int slot, const float (&v)[32]) const {
    const int lane = threadIdx.x & 31;
    uint8_t* row = reinterpret_cast<uint8_t*>(slots + slot * SF) + lane * 64;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint4 q;
      __half2 h0 = __floats2half2_rn(v[8 * j], v[8 * j + 1]);
      __half2 h1 = __floats2half2_rn(v[8 * j + 2], v[8 * j + 3]);
      __half2 h2 = __floats2half2_rn(v[8 * j + 4], v[8 * j + 5]);
      __half2 h3 = __floats2half2_rn(v[8 * j + 6], v[8 * j + 7]);
      q.x = *reinterpret_cast<uint32_t*>(&h0);
      q.y = *reinterpret_cast<uint32_t*>(&h1);
      q.z = *reinterpret_cast<uint32_t*>(&h2);
      q.w = *reinterpret_cast<uint32_t*>(&h3);
      *reinterpret_cast<uint4*>(row + ((j ^ ((lane >> 1) & 3)) << 4)) = q;
    }
  }
  __device__ __forceinline__ void in_h(int slot, float (&v)[32]) const {
    const int lane = threadIdx.x & 31;
    const uint8_t* row = reinterpret_cast<const uint8_t*>(slots + (ib + slot) * SF) + lane * 64;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint4 q = *reinterpret_cast<const uint4*>(row + ((j ^ ((lane >> 1) & 3)) << 4));
      const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w[u]));
        v[8 * j + 2 * u] = f.x;
        v[8 * j + 2 * u + 1] = f.y;
      }
    }
  }
  __device__ __forceinline__ void put_h(int map, const float (&v)[32], int c2, int c3) {
    const int slot = *next;
    *next = slot + 1 == NS ? 0 : slot + 1;
    if ((threadIdx.x & 31) == 0) bulk_wait_read<NS - 1>();
    __syncwarp();
    write_row_h(slot, v);
    issue(slot, map, c2, c3);
  }
  __device__ __forceinline__ void put_at_h(int slot, int map, const float (&v)[32], int c2,
                                           int c3) {
    write_row_h(ib + slot, v);
    issue(ib + slot, map, c2, c3);
  }
  // store v (this thread's row) to map at (n0, m0, c2, c3) through the ring
  __device__ __forceinline__ void put(int map, const float (&v)[32], int c2, int c3) {
    const int slot = *next;
    *next = slot + 1 == NS ? 0 : slot + 1;
    if ((threadIdx.x & 31) == 0) bulk_wait_read<NS - 1>();
    __syncwarp();
    write_row(slot, v);
    issue(slot, map, c2, c3);
  }
  // store v through input slot `slot` (already consumed by this thread's row)
  __device__ __forceinline__ void put_at(int slot, int map, const float (&v)[32], int c2, int c3) {
    write_row(ib + slot, v);
    issue(ib + slot, map, c2, c3);
  }
};

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

constexpr int kTcBiasWarps = 4;
__host__ __device__ constexpr int tc_threads(bool bias, int ew = 8) {
  return 32 * (2 + ew + (bias ? kTcBiasWarps : 0));
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Persistent, warp-specialised tcgen05 GEMM.  CTAs walk tiles t = blockIdx.x,
// blockIdx.x + gridDim.x, ... (tn fastest, then tm, then batch/split z).
//   warp 0      TMA producer over all k-blocks of all its tiles (kTcStages ring)
//   warp 1      TMEM allocator + single-thread MMA issuer; accumulator double
//               buffered in TMEM so tile t's epilogue overlaps tile t+1's MMAs
//   warps 2..9  epilogue (two per TMEM lane quadrant, alternating 32-column
//               chunks): tcgen05.ld -> fused epilogue -> global
//   warps 10-13 (BIAS only) column sums of the B tile of every k-block of
//               the tiles with tm == 0, read straight from the smem ring
// CL = 2: CTA pairs (clusters of 2 along x) own m-tiles 2p and 2p+1 of the
// same (tn, z); each CTA TMA-multicasts one half of the shared B tile to
// both, so per-SM operand traffic per k-block drops from A+B to A+B/2.
// Stage reuse then needs both CTAs' MMA commits (and bias reads).
template <int BN, bool AMN, bool BMN, bool BIAS, class Epi, int ZIN = 1, int CL = 1, int EW = 8,
          bool H = false>
__global__ void __launch_bounds__(tc_threads(BIAS, EW), 1)
k_tc_gemm(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
          const __grid_constant__ CUtensorMap tma_c, const __grid_constant__ CUtensorMap tma_d,
          TcShape s, Epi epi) {
  static_assert(!BIAS || BMN, "fused bias sums read an MN-major B tile");
  static_assert(!H || !BMN || BN % 64 == 0, "fp16 MN-major B boxes are 64 wide");
  constexpr int BK = tc_bk<H>();
  static_assert(ZIN == 1 || !BIAS, "multi-branch tiles have no fused bias");
  static_assert(TcSmem<BN, ZIN>::kCols <= 512, "TMEM holds 512 columns");
  constexpr bool TS = EpiTmaStore<Epi>::value;
  constexpr int kTsSlots = TS ? EpiTsSlots<Epi>::value : 0;
  constexpr int kTsSB = EpiTsSlotBytes<Epi>::value;
  constexpr int kTsIn = EpiTsIn<Epi>::value;
  static_assert(kTsIn == 0 || 2 * kTsIn == kTsSlots,
                "input boxes are double-buffered in the TMA-store slots");
  static_assert(2 * (kStagesMax + 2 + 2 + EW) * 8 <= 512, "barrier area");
  constexpr bool TR = ZIN > 1 || EpiTransposed<Epi>::value;  // also the !s.ts fallback
  constexpr int kTcEpiWarps = EW;  // epilogue warps: EW / 4 per TMEM lane quadrant
  static_assert(EW % 4 == 0, "whole TMEM lane quadrants per epilogue warp group");
  extern __shared__ uint8_t smem_raw[];
  using SM = TcSmem<BN, ZIN, TR, EW, kTsSlots, kTsSB>;
  uint8_t* smem = reinterpret_cast<uint8_t*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  constexpr int kStages = SM::kStages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + SM::kBarOffset);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  uint64_t* wbar = tempty + 4;  // 2 per epilogue warp: its double-buffered TMA-loaded input boxes

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n_tn = s.N / BN;
  const int n_tm = (s.M + kTcBM - 1) / kTcBM;
  const int nzt = (ZIN > 1 ? 1 : s.nzb) * (s.kmode == 0 ? 1 : s.nsplit);
  const int crank = CL > 1 ? (int)cluster_rank() : 0;
  const int n_tmu = n_tm / CL;               // m-tile units (pairs when CL = 2)
  const int n_tiles = n_tn * n_tmu * nzt;    // work units
  const int u0 = blockIdx.x / CL, ustride = gridDim.x / CL;
  constexpr uint16_t kMask = (uint16_t)((1u << CL) - 1u);

  auto tile_coords = [&](int t, int& tn, int& tm, int& zb, int& zg, int& kb0, int& nkb) {
    tn = t % n_tn;
    const int r = t / n_tn;
    tm = (r % n_tmu) * CL + crank;
    const int z = r / n_tmu;
    const int nzb = ZIN > 1 ? 1 : s.nzb;
    zb = z % nzb;
    zg = z / nzb;
    int k_begin = 0, k_end = s.K;
    if (s.kmode == 1) {
      k_begin = group_begin(s.g0 + zg, s.B_global) - s.lane0;
      k_end = group_begin(s.g0 + zg + 1, s.B_global) - s.lane0;
    } else if (s.kmode == 2) {
      const int chunk = s.K / s.nsplit;
      k_begin = zg * chunk;
      k_end = k_begin + chunk;
    }
    kb0 = k_begin;
    nkb = (k_end - k_begin) / BK;
  };

  if (warp == 0 && lane == 0) {
    // descriptors fetched while the predecessor drains (before pdl_entry)
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tma_a) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tma_b) : "memory");
    if (s.ts) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tma_c) : "memory");
      if (kTsIn > 0) asm volatile("prefetch.tensormap [%0];" ::"l"(&tma_d) : "memory");
    }
    for (int st = 0; st < kStages; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], CL * (BIAS ? 2 : 1));
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kTcEpiWarps);
    }
    if constexpr (kTsIn > 0)
      for (int w = 0; w < 2 * kTcEpiWarps; ++w) mbar_init(&wbar[w], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(SM::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  if (CL > 1) cluster_sync_all();  // peer barriers initialised before any multicast
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_entry();  // after the TMEM allocation (see common.cuh)

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer
      int it = 0;
      for (int t = u0; t < n_tiles; t += ustride) {
        int tn, tm, zb, zg, kb0, nkb;
        tile_coords(t, tn, tm, zb, zg, kb0, nkb);
        const int n0 = tn * BN, m0 = tm * kTcBM;
        for (int q = 0; q < nkb * s.nsum; ++q, ++it) {
          const int st = it % kStages;
          const uint32_t ph = (uint32_t)(it / kStages) & 1u;
          mbar_wait(&empty[st], ph ^ 1u);
          // summed sub-problems (kBatchSum: the MBRB branches of the branch
          // dgrad) interleave per k-block -- branch 0 then branch 1 of each
          // 64-deep block, the order of the fused MBRB backward (mbrb_fused.cuh)
          const int sub = q % s.nsum;
          const int k = kb0 + (q / s.nsum) * BK;
          const int az = s.a_batch == kBatchZ ? zb : (s.a_batch == kBatchSum ? sub : 0);
          const int bz = s.b_batch == kBatchZ ? zb : (s.b_batch == kBatchSum ? sub : 0);
          uint8_t* sa = smem + st * SM::kStageBytes;
          uint8_t* sb = sa + SM::kABytes;
          mbar_expect_tx(&full[st], SM::kStageBytes);
          if (AMN) {
            constexpr int kW = H ? 64 : 32;  // MN width of one box
#pragma unroll
            for (int j = 0; j < kTcBM / kW; ++j)
              tma_load_3d(sa + j * kW * 128, &tma_a, &full[st], m0 + kW * j, k, az);
          } else {
            tma_load_3d(sa, &tma_a, &full[st], k, m0, az);
          }
#pragma unroll
          for (int zi = 0; zi < ZIN; ++zi) {
            const int bzz = ZIN > 1 ? zi : bz;
            uint8_t* sbz = sb + zi * SM::kBBytes;
            constexpr int kW = H ? 64 : 32;
            if constexpr (CL == 1) {
              if (BMN) {
#pragma unroll
                for (int j = 0; j < BN / kW; ++j)
                  tma_load_3d(sbz + j * kW * 128, &tma_b, &full[st], n0 + kW * j, k, bzz);
              } else {
                tma_load_3d(sbz, &tma_b, &full[st], k, n0, bzz);
              }
            } else {
              // this CTA's half of B, multicast into both CTAs of the pair
              if (BMN) {
                constexpr int nb = BN / kW / CL > 0 ? BN / kW / CL : 1;
#pragma unroll
                for (int jj = 0; jj < nb; ++jj) {
                  const int j = crank * nb + jj;
                  tma_load_3d_mc(sbz + j * kW * 128, &tma_b, &full[st], n0 + kW * j, k, bzz,
                                 kMask);
                }
              } else {
                constexpr int rows = BN / CL;
                tma_load_3d_mc(sbz + crank * rows * 128, &tma_b, &full[st], k, n0 + crank * rows,
                               bzz, kMask);
              }
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer
      constexpr uint32_t idesc = H ? idesc_f16(kTcBM, BN, AMN ? 1 : 0, BMN ? 1 : 0)
                                   : idesc_tf32(kTcBM, BN, AMN ? 1 : 0, BMN ? 1 : 0);
      const uint32_t mlbo = s.mn_lbo ? (uint32_t)s.mn_lbo : kMnH_LBO;
      const uint32_t msbo = s.mn_sbo ? (uint32_t)s.mn_sbo : kMnH_SBO;
      int it = 0, lt = 0;
      for (int t = u0; t < n_tiles; t += ustride, ++lt) {
        int tn, tm, zb, zg, kb0, nkb;
        tile_coords(t, tn, tm, zb, zg, kb0, nkb);
        const int acc = lt & 1;
        mbar_wait(&tempty[acc], (((uint32_t)lt >> 1) & 1u) ^ 1u);
        tc_fence_after();
        const uint32_t dtm = tmem + (uint32_t)(acc * ZIN * BN);
        const int nq = nkb * s.nsum;
        for (int q = 0; q < nq; ++q, ++it) {
          const int st = it % kStages;
          const uint32_t ph = (uint32_t)(it / kStages) & 1u;
          mbar_wait(&full[st], ph);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + st * SM::kStageBytes);
#pragma unroll
          for (int zi = 0; zi < ZIN; ++zi) {
            const uint32_t sb = sa + SM::kABytes + zi * SM::kBBytes;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              if constexpr (H) {
                const uint64_t ad = AMN ? sdesc(sa + kk * 2048, mlbo, msbo, kLayoutSW128)
                                        : sdesc(sa + kk * 32, 16, 1024, kLayoutSW128);
                const uint64_t bd = BMN ? sdesc(sb + kk * 2048, mlbo, msbo, kLayoutSW128)
                                        : sdesc(sb + kk * 32, 16, 1024, kLayoutSW128);
                tc_mma_f16(dtm + (uint32_t)(zi * BN), ad, bd, idesc, (q > 0 || kk > 0) ? 1u : 0u);
              } else {
                const uint64_t ad = AMN ? sdesc(sa + kk * 1024, 4096, 512, kLayoutSW128Base32B)
                                        : sdesc(sa + kk * 32, 16, 1024, kLayoutSW128);
                const uint64_t bd = BMN ? sdesc(sb + kk * 1024, 4096, 512, kLayoutSW128Base32B)
                                        : sdesc(sb + kk * 32, 16, 1024, kLayoutSW128);
                tc_mma_tf32(dtm + (uint32_t)(zi * BN), ad, bd, idesc,
                            (q > 0 || kk > 0) ? 1u : 0u);
              }
            }
          }
          if constexpr (CL == 1)
            tc_commit(&empty[st]);
          else
            tc_commit_mc(&empty[st], kMask);
        }
        tc_commit(&tfull[acc]);
      }
    }
  } else if (warp < 2 + kTcEpiWarps) {
    // ---------------- epilogue warps (TMEM lane quadrant = warp % 4)
    const int quad = warp & 3;
    const int half = (warp - 2) >> 2;  // which of the EW/4 warps of this quadrant
    int lt = 0;
    int ts_next = 0;       // TMA-store box ring position
    uint32_t ts_wph = 0;   // phases of this warp's two input-box barriers (bit = slot pair)
    int ts_pair = 0;       // slot pair holding the current block's input boxes
    float* const ts_slots = reinterpret_cast<float*>(smem + SM::kEpiOffset) +
                            (warp - 2) * (kTsSlots > 0 ? kTsSlots : 1) * (kTsSB / 4);
    // TMA loads of the input boxes of block (tile tq, column cq) into slot pair `pair`
    auto ts_issue = [&](int tq, int cq, int pair) {
      if constexpr (kTsIn > 0) {
        int tn, tm, zb, zg, kb0, nkb;
        tile_coords(tq, tn, tm, zb, zg, kb0, nkb);
        uint64_t* bar = &wbar[(warp - 2) * 2 + pair];
        mbar_expect_tx(bar, kTsIn * EpiTsInBytes<Epi>::value);
#pragma unroll
        for (int i = 0; i < kTsIn; ++i) {
          int c2, c3;
          epi.ts_in(i, zb, zg, c2, c3);
          tma_load_4d(ts_slots + (pair * kTsIn + i) * (kTsSB / 4), &tma_d, bar,
                      tn * BN + cq, tm * kTcBM + quad * 32, c2, c3);
        }
      }
    };
    if constexpr (TS && kTsIn > 0) {
      if (s.ts && lane == 0 && u0 < n_tiles) ts_issue(u0, half * 32, 0);
    }
    for (int t = u0; t < n_tiles; t += ustride, ++lt) {
      int tn, tm, zb, zg, kb0, nkb;
      tile_coords(t, tn, tm, zb, zg, kb0, nkb);
      const int acc = lt & 1;
      const int n0 = tn * BN;
      const int m = tm * kTcBM + quad * 32 + lane;
      const bool any = nkb * s.nsum > 0;
      mbar_wait(&tfull[acc], ((uint32_t)lt >> 1) & 1u);
      tc_fence_after();
      float* T = reinterpret_cast<float*>(smem + SM::kEpiOffset) + (warp - 2) * ZIN * kTcTileFloats;
      const int m_base = tm * kTcBM + quad * 32;
#pragma unroll 1
      for (int c = half * 32; c < BN; c += 32 * (EW / 4)) {
        if (s.dbg == 3) continue;  // microbenchmark ablation: no epilogue at all
        if constexpr (TS) {
          if (s.ts) {
            float* slots = ts_slots;
            if constexpr (kTsIn > 0) {
              // this block's inputs were issued one block ahead; now issue the
              // next block's (this warp's next column, or its next tile's first)
              // into the other slot pair, whose stores must have read it
              int tq = t, cq = c + 32 * (EW / 4);
              if (cq >= BN) {
                tq = t + ustride;
                cq = half * 32;
              }
              if (lane == 0) {
                bulk_wait_read<0>();
                if (tq < n_tiles) ts_issue(tq, cq, ts_pair ^ 1);
              }
            }
            float v[ZIN][32];
#pragma unroll
            for (int zi = 0; zi < ZIN; ++zi) {
              if (any) {
                tmem_ld32(tmem + ((uint32_t)(quad * 32) << 16) +
                              (uint32_t)((acc * ZIN + zi) * BN + c),
                          v[zi]);
              } else {
#pragma unroll
                for (int j = 0; j < 32; ++j) v[zi][j] = 0.f;
              }
              if (s.dbg == 1) {
#pragma unroll
                for (int j = 0; j < 32; ++j) v[zi][j] = (float)(m * 1000 + n0 + c + j);
              }
            }
            int ib = 0;
            if constexpr (kTsIn > 0) {
              mbar_wait(&wbar[(warp - 2) * 2 + ts_pair], (ts_wph >> ts_pair) & 1u);
              ts_wph ^= 1u << ts_pair;
              ib = ts_pair * kTsIn;
              ts_pair ^= 1;
            }
            TsIo<kTsSlots, kTsSB / 4> io{slots, {&tma_c, &tma_d}, n0 + c, m_base, &ts_next, ib};
            epi.ts_chunk(io, zb, zg, m, n0 + c, v);
            continue;
          }
        }
        if constexpr (!TR) {
          float v[32];
          if (any) {
            tmem_ld32(tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(acc * BN + c), v);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = 0.f;
          }
          if (s.dbg == 1) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = (float)(m * 1000 + n0 + c + j);
          }
          if (s.dbg == 2) {  // microbenchmark ablation: TMEM loads only
            float x = 0.f;
#pragma unroll
            for (int j = 0; j < 32; ++j) x += v[j];
            if (x == 12345.678f) epi.row32(zb, zg, m, n0 + c, v);
            continue;
          }
          if (m < s.M) epi.row32(zb, zg, m, n0 + c, v);
        } else {
#pragma unroll
          for (int zi = 0; zi < ZIN; ++zi) {
            float v[32];
            if (any) {
              tmem_ld32(tmem + ((uint32_t)(quad * 32) << 16) +
                            (uint32_t)((acc * ZIN + zi) * BN + c),
                        v);
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] = 0.f;
            }
            if (s.dbg == 1) {
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] = (float)(m * 1000 + n0 + c + j);
            }
#pragma unroll
            for (int j = 0; j < 32; ++j) T[zi * kTcTileFloats + lane * 32 + (j ^ lane)] = v[j];
          }
          __syncwarp();
          if (m_base < s.M) {
            if constexpr (ZIN == 1)
              epi.tile(T, zb, zg, m_base, n0 + c, s.M);
            else
              epi.tile_z(T, m_base, n0 + c, s.M);
          }
          __syncwarp();
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
    if constexpr (TS) {
      if (s.ts && lane == 0) bulk_wait_all();
    }
  } else if (BIAS) {
    // ---------------- bias warps: column sums of B over this tile's K range
    const int bt = threadIdx.x - 32 * (2 + kTcEpiWarps);  // 0..127
    // columns per thread (fp16: column pairs)
    constexpr int kCols = (H ? BN / 2 : BN) / (32 * kTcBiasWarps) > 0
                              ? (H ? BN / 2 : BN) / (32 * kTcBiasWarps)
                              : 1;
    auto bias_col = [&](int j) { return H ? 2 * (bt + j * 32 * kTcBiasWarps)
                                          : bt + j * 32 * kTcBiasWarps; };
    int it = 0;
    for (int t = u0; t < n_tiles; t += ustride) {
      int tn, tm, zb, zg, kb0, nkb;
      tile_coords(t, tn, tm, zb, zg, kb0, nkb);
      const bool do_sum = tm == 0 && s.bias_part != nullptr;
      float sum[kCols], sum2[kCols];  // sum2: second column of an fp16 pair
#pragma unroll
      for (int j = 0; j < kCols; ++j) sum[j] = sum2[j] = 0.f;
      const int nq = nkb * s.nsum;
      for (int q = 0; q < nq; ++q, ++it) {
        const int st = it % kStages;
        const uint32_t ph = (uint32_t)(it / kStages) & 1u;
        mbar_wait(&full[st], ph);
        if (do_sum) {
          const uint8_t* sb = smem + st * SM::kStageBytes + SM::kABytes;
#pragma unroll
          for (int j = 0; j < kCols; ++j) {
            const int n = bias_col(j);
            if (n < BN) {
              if constexpr (H) {
                // fp16 MN-major: 64-wide boxes of 64 K-rows, 16-byte chunk c of
                // row k at c ^ (k & 7) (SWIZZLE_128B); this thread's column
                // pair (n, n + 1) is one half2 per row
                // (32-bit shared addresses: LDS with immediate offsets, not
                // generic 64-bit loads -- these warps gate every stage's release)
                const int box = n >> 6, nn = n & 63, chunk = nn >> 3;
                const uint32_t base = smem_u32(sb + box * 8192 + (nn & 7) * 2);
                float s0 = 0.f, s1 = 0.f;
#pragma unroll 8
                for (int k = 0; k < BK; ++k) {
                  uint32_t w;
                  asm volatile("ld.shared.b32 %0, [%1];"
                               : "=r"(w)
                               : "r"(base + (uint32_t)(k * 128 + ((chunk ^ (k & 7)) << 4))));
                  const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w));
                  s0 += f.x;
                  s1 += f.y;
                }
                sum[j] += s0;
                sum2[j] += s1;
              } else {
                const int box = n >> 5, nn = n & 31, chunk = nn >> 3;
                const uint32_t base = smem_u32(sb + box * 4096) + (uint32_t)(nn & 7) * 4u;
#pragma unroll 8
                for (int k = 0; k < kTcBK; ++k) {
                  float v;
                  asm volatile("ld.shared.f32 %0, [%1];"
                               : "=f"(v)
                               : "r"(base + (uint32_t)(k * 128 + ((chunk ^ (k & 3)) << 5))));
                  sum[j] += v;
                }
              }
            }
          }
        }
        named_bar(1, 32 * kTcBiasWarps);
        if (bt == 0) {
          if constexpr (CL == 1) {
            mbar_arrive(&empty[st]);
          } else {
#pragma unroll
            for (int r = 0; r < CL; ++r) mbar_arrive_cluster(&empty[st], (uint32_t)r);
          }
        }
      }
      if (do_sum) {
#pragma unroll
        for (int j = 0; j < kCols; ++j) {
          const int n = bias_col(j);
          float* dst = s.bias_part + (int64_t)(s.g0 + zg) * s.bias_gstride + s.bias_off +
                       zb * s.bias_zstride + tn * BN + n;
          if (n < BN && tn * BN + n < s.N) dst[0] = sum[j];
          if (H && n + 1 < BN && tn * BN + n + 1 < s.N) dst[1] = sum2[j];
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (CL > 1) cluster_sync_all();  // no CTA leaves while its peer may still signal it
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(SM::kTmemCols));
  }
}

// ------------------------------------------------------- host: tensor maps

// cuTensorMapEncodeTiled through the runtime's driver entry point, so the
// library does not link libcuda (it must load on CPU-only hosts).
typedef CUresult (*PfnEncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline PfnEncodeTiled encode_tiled_fn() {
  static PfnEncodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PfnEncodeTiled>(p);
  }
  return fn;
}

// 3-D fp32 tensor map: dims {inner, rows, batch}; strides in elements.
// kind: bit 0 = MN-major, bit 1 = fp16 elements
inline int make_tmap(CUtensorMap* map, const void* base, uint64_t inner, uint64_t rows,
                     uint64_t batch, uint64_t row_stride, uint64_t batch_stride, uint32_t box_inner,
                     uint32_t box_rows, int kind) {
  const bool mn_major = kind & 1, half = kind & 2;
  const uint64_t es = half ? 2 : 4;
  cuuint64_t dims[3] = {inner, rows, batch < 1 ? 1 : batch};
  cuuint64_t strides[2] = {row_stride * es, (batch_stride ? batch_stride : row_stride * rows) * es};
  cuuint32_t box[3] = {box_inner, box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  PfnEncodeTiled enc = encode_tiled_fn();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled entry point unavailable");
    return EDPC_ERR_CUDA;
  }
  CUresult r = enc(map, half ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                   3, (void*)base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   (mn_major && !half) ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B
                                       : CU_TENSOR_MAP_SWIZZLE_128B,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed with CUresult " + std::to_string((int)r));
    return EDPC_ERR_CUDA;
  }
  return EDPC_OK;
}

// Output map of a TMA-store epilogue: 4D fp32, box 32 x 32 x 1 x 1, 128B
// swizzle.  False when TMA cannot address it (16-byte alignment of the base
// and of every stride); the kernel then stores with row32.
inline bool make_store_tmap(CUtensorMap* map, const TcStoreMap& d) {
  if (((uintptr_t)d.base & 15) != 0 || d.dims[0] < 32) return false;
  const uint64_t es = d.half ? 2 : 4;
  cuuint64_t dims[4] = {d.dims[0], d.dims[1], d.dims[2] ? d.dims[2] : 1, d.dims[3] ? d.dims[3] : 1};
  cuuint64_t strides[3];
  uint64_t prev = d.dims[0];
  for (int i = 0; i < 3; ++i) {
    uint64_t st = d.strides[i];
    if (dims[i + 1] == 1 || st == 0) st = prev;  // unused dimension: any valid stride
    if ((st * es) % 16 != 0 || st * es >= (1ull << 40)) return false;
    strides[i] = st * es;
    prev = st * dims[i + 1];
  }
  cuuint32_t box[4] = {32, 32, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  PfnEncodeTiled enc = encode_tiled_fn();
  if (!enc) return false;
  return enc(map, d.half ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4,
             (void*)d.base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             d.half ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

struct StoreTmapCache {
  std::mutex mu;
  std::map<std::tuple<const void*, uint64_t, uint64_t, uint64_t, uint64_t, uint64_t, uint64_t,
                      uint64_t, int>,
           std::pair<bool, CUtensorMap>>
      maps;
  bool get(CUtensorMap* out, const TcStoreMap& d) {
    auto key = std::make_tuple((const void*)d.base, d.dims[0], d.dims[1], d.dims[2], d.dims[3],
                               d.strides[0], d.strides[1], d.strides[2], d.half);
    std::lock_guard<std::mutex> g(mu);
    auto it = maps.find(key);
    if (it == maps.end()) {
      CUtensorMap m{};
      bool ok = make_store_tmap(&m, d);
      it = maps.emplace(key, std::make_pair(ok, m)).first;
    }
    *out = it->second.second;
    return it->second.first;
  }
};

inline StoreTmapCache& store_tmap_cache() {
  static StoreTmapCache c;
  return c;
}

// Both maps of a TMA-store epilogue (a null base = unused); 1 if usable.
template <class Epi>
inline int ts_maps(const Epi& epi, const TcShape& s, CUtensorMap& tc, CUtensorMap& td) {
  TcStoreMap c{}, d{};
  if (!epi.store_maps(s, c, d)) return 0;
  if (!store_tmap_cache().get(&tc, c)) return 0;
  if (d.base && !store_tmap_cache().get(&td, d)) return 0;
  return 1;
}

// An operand as stored in global memory: row-major [rows][inner] (+ batch).
struct TcOperand {
  const void* ptr;  // fp32, or fp16 on the H path
  int64_t ld;      // row stride (elements)
  int64_t sbatch;  // batch stride (elements), 0 if no batch
  int nbatch;
};

struct TmapCache {
  std::mutex mu;
  std::map<std::tuple<const void*, uint64_t, uint64_t, uint64_t, uint64_t, uint64_t, uint32_t,
                      uint32_t, int>,
           CUtensorMap>
      maps;
  int get(CUtensorMap* out, const void* base, uint64_t inner, uint64_t rows, uint64_t batch,
          uint64_t ld, uint64_t sb, uint32_t bi, uint32_t br, int mn) {
    auto key = std::make_tuple((const void*)base, inner, rows, batch, ld, sb, bi, br, mn);
    std::lock_guard<std::mutex> g(mu);
    auto it = maps.find(key);
    if (it != maps.end()) {
      *out = it->second;
      return EDPC_OK;
    }
    CUtensorMap m;
    int r = make_tmap(&m, base, inner, rows, batch, ld, sb, bi, br, mn);
    if (r != EDPC_OK) return r;
    maps.emplace(key, m);
    *out = m;
    return EDPC_OK;
  }
};

inline TmapCache& tmap_cache() {
  static TmapCache c;
  return c;
}

// True when the shape tiles cleanly: M any (TMA zero-fills, epilogue masks),
// N a multiple of 32 (<= 256 per tile or a multiple of 256), K chunks of 32.
inline bool tc_shape_ok(int N, int Kchunk) {
  if (N % 32 != 0 || Kchunk % kTcBK != 0 || Kchunk <= 0) return false;
  return N <= 256 ? (N == 32 || N == 64 || N == 128 || N == 256) : (N % 256 == 0);
}

inline int num_sms() {
  static int n[16] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 16 && !n[dev]) cudaDeviceGetAttribute(&n[dev], cudaDevAttrMultiProcessorCount, dev);
  return dev < 16 && n[dev] ? n[dev] : 148;
}

// 2-CTA multicast clusters (CL = 2): measured slower than CL = 1 in round 1
// (the GEMMs were not L2-bandwidth bound), and under the round-2 schedule
// (programmatic dependent launch on every step kernel, fused cluster MBRB
// kernels beside them) the CL = 2 step deadlocks, so the path is compiled out
// of the launch decision until it is reworked; the kernel template keeps it.
inline constexpr bool cluster_enabled() { return false; }

template <typename Kern, typename Epi>
inline cudaError_t launch_tc(Kern kern, int grid, int threads, int smem, cudaStream_t st, int cl,
                             const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tc,
                             const CUtensorMap& td, const TcShape& s, const Epi& epi) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)threads);
  cfg.dynamicSmemBytes = (size_t)smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, kern, ta, tb, tc, td, s, epi);
}

template <typename Kern>
inline void set_smem_attr(Kern kern, int bytes, bool& done) {
  if (!done) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    done = true;
  }
}

// TMA maps of the two operands.  A: K-major -> [M rows][K inner]; MN-major ->
// [K rows][M inner].  B: K-major -> [N rows][K inner] (box BN/cl rows);
// MN-major -> [K rows][N inner].  fp32 boxes are 32 elements (128 B) wide,
// fp16 boxes 64; MN-major boxes are square.
template <int BN, bool AMN, bool BMN, bool H>
inline int tc_operand_maps(const TcShape& s, const TcOperand& A, const TcOperand& B, int cl,
                           CUtensorMap& ta, CUtensorMap& tb) {
  constexpr uint32_t W = tc_bk<H>();
  constexpr int kh = H ? 2 : 0;
  int r;
  if (AMN)
    r = tmap_cache().get(&ta, A.ptr, (uint64_t)s.M, (uint64_t)s.K, (uint64_t)A.nbatch,
                         (uint64_t)A.ld, (uint64_t)A.sbatch, W, W, 1 | kh);
  else
    r = tmap_cache().get(&ta, A.ptr, (uint64_t)s.K, (uint64_t)s.M, (uint64_t)A.nbatch,
                         (uint64_t)A.ld, (uint64_t)A.sbatch, W, kTcBM, kh);
  if (r != EDPC_OK) return r;
  if (BMN)
    r = tmap_cache().get(&tb, B.ptr, (uint64_t)s.N, (uint64_t)s.K, (uint64_t)B.nbatch,
                         (uint64_t)B.ld, (uint64_t)B.sbatch, W, W, 1 | kh);
  else
    r = tmap_cache().get(&tb, B.ptr, (uint64_t)s.K, (uint64_t)s.N, (uint64_t)B.nbatch,
                         (uint64_t)B.ld, (uint64_t)B.sbatch, W, BN / cl, kh);
  return r;
}

template <int BN, bool AMN, bool BMN, bool H = false, class Epi>
inline int tc_launch(const TcShape& s, const TcOperand& A, const TcOperand& B, const Epi& epi,
                     cudaStream_t st) {
  constexpr bool kTS = EpiTmaStore<Epi>::value;
  constexpr int kSmem =
      TcSmem<BN, 1, EpiTransposed<Epi>::value, 8, kTS ? EpiTsSlots<Epi>::value : 0,
             EpiTsSlotBytes<Epi>::value>::kBytes;
  const int n_tm = cdiv(s.M, kTcBM);
  const int cl = (cluster_enabled() && n_tm % 2 == 0) ? 2 : 1;
  CUtensorMap ta, tb, tc{}, td{};
  TcShape s2 = s;
  if constexpr (kTS) s2.ts = ts_maps(epi, s, tc, td);
  if (EpiRequireTs<Epi>::value && !s2.ts) {
    set_error("tc_gemm: epilogue output not addressable by TMA (alignment)");
    return EDPC_ERR_INVALID;
  }
  int r;
  r = tc_operand_maps<BN, AMN, BMN, H>(s, A, B, cl, ta, tb);
  if (r != EDPC_OK) return r;
  const int nz = s.nzb * (s.kmode == 0 ? 1 : s.nsplit);
  const int units = (s.N / BN) * (n_tm / cl) * nz;
  const int max_units = num_sms() / cl;
  const int grid = (units < max_units ? units : max_units) * cl;
  int dev = 0;
  cudaGetDevice(&dev);
  const int di = dev < 16 ? dev : 0;
  cudaError_t e = cudaSuccess;
  bool launched = false;
  if constexpr (BMN) {
    if (s.bias_part) {
      if (cl == 2) {
        static bool done[16] = {};
        auto kern = k_tc_gemm<BN, AMN, BMN, true, Epi, 1, 2, 8, H>;
        set_smem_attr(kern, kSmem, done[di]);
        e = launch_tc(kern, grid, tc_threads(true), kSmem, st, 2, ta, tb, tc, td, s2, epi);
      } else {
        static bool done[16] = {};
        auto kern = k_tc_gemm<BN, AMN, BMN, true, Epi, 1, 1, 8, H>;
        set_smem_attr(kern, kSmem, done[di]);
        e = launch_tc(kern, grid, tc_threads(true), kSmem, st, 1, ta, tb, tc, td, s2, epi);
      }
      launched = true;
    }
  }
  if (!launched) {
    if (cl == 2) {
      static bool done[16] = {};
      auto kern = k_tc_gemm<BN, AMN, BMN, false, Epi, 1, 2, 8, H>;
      set_smem_attr(kern, kSmem, done[di]);
      e = launch_tc(kern, grid, tc_threads(false), kSmem, st, 2, ta, tb, tc, td, s2, epi);
    } else {
      static bool done[16] = {};
      auto kern = k_tc_gemm<BN, AMN, BMN, false, Epi, 1, 1, 8, H>;
      set_smem_attr(kern, kSmem, done[di]);
      e = launch_tc(kern, grid, tc_threads(false), kSmem, st, 1, ta, tb, tc, td, s2, epi);
    }
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("k_tc_gemm launch: ") + cudaGetErrorString(e));
    return EDPC_ERR_CUDA;
  }
  return EDPC_OK;
}

// Multi-branch launch: ZIN branch GEMMs sharing A, one CTA per (tm, tn).
template <int BN, int ZIN, bool BMN, bool H = false, class Epi>
inline int tc_launch_zin(const TcShape& s, const TcOperand& A, const TcOperand& B,
                         const Epi& epi, cudaStream_t st) {
  // the transposed fused-GeLU epilogue is issue-bound (16 epilogue warps);
  // the TMA-store form keeps its registers with 8
  constexpr bool kTS = EpiTmaStore<Epi>::value;
  constexpr int kZinEW = (!kTS && BN % 128 == 0) ? 16 : 8;
  constexpr int kSmem = TcSmem<BN, ZIN, true, kZinEW, kTS ? EpiTsSlots<Epi>::value : 0,
                               EpiTsSlotBytes<Epi>::value>::kBytes;
  const int n_tm = cdiv(s.M, kTcBM);
  const int cl = (cluster_enabled() && n_tm % 2 == 0) ? 2 : 1;
  CUtensorMap ta, tb;
  int r = tc_operand_maps<BN, false, BMN, H>(s, A, B, cl, ta, tb);
  if (r != EDPC_OK) return r;
  CUtensorMap tc{}, td{};
  TcShape s2 = s;
  if constexpr (kTS) s2.ts = ts_maps(epi, s, tc, td);
  if (EpiRequireTs<Epi>::value && !s2.ts) {
    set_error("tc_gemm: epilogue output not addressable by TMA (alignment)");
    return EDPC_ERR_INVALID;
  }
  const int units = (s.N / BN) * (n_tm / cl);
  const int max_units = num_sms() / cl;
  const int grid = (units < max_units ? units : max_units) * cl;
  int dev = 0;
  cudaGetDevice(&dev);
  const int di = dev < 16 ? dev : 0;
  cudaError_t e;
  if (cl == 2) {
    static bool done[16] = {};
    auto kern = k_tc_gemm<BN, false, BMN, false, Epi, ZIN, 2, kZinEW, H>;
    set_smem_attr(kern, kSmem, done[di]);
    e = launch_tc(kern, grid, tc_threads(false, kZinEW), kSmem, st, 2, ta, tb, tc, td, s2, epi);
  } else {
    static bool done[16] = {};
    auto kern = k_tc_gemm<BN, false, BMN, false, Epi, ZIN, 1, kZinEW, H>;
    set_smem_attr(kern, kSmem, done[di]);
    e = launch_tc(kern, grid, tc_threads(false, kZinEW), kSmem, st, 1, ta, tb, tc, td, s2, epi);
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("k_tc_gemm<zin> launch: ") + cudaGetErrorString(e));
    return EDPC_ERR_CUDA;
  }
  return EDPC_OK;
}

// BN dispatch: the widest tile <= 256 that divides N
inline int bn_cap() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("EDPC_BN_MAX");  // tuning knob (tests / microbenchmarks)
    v = e ? atoi(e) : 256;
  }
  return v;
}

template <bool AMN, bool BMN, bool H = false, class Epi>
inline int tc_gemm(const TcShape& s, const TcOperand& A, const TcOperand& B, const Epi& epi,
                   cudaStream_t st) {
  // Tile width: the widest BN whose tile count still fills 3/4 of the SMs;
  // small GEMMs (head, LTE projections, their weight gradients: 8-32 tiles
  // at BN 256) are bound by per-SM TMA bandwidth and latency, so they trade
  // MMA width for CTAs.
  const int cap = bn_cap();
  const int nz = s.nzb * (s.kmode == 0 ? 1 : s.nsplit);
  const int n_tm = cdiv(s.M, kTcBM);
  const int want = num_sms() * 3 / 4;
  int bn = 0;
  for (int c : {256, 128, 64, 32}) {
    if (c > cap || s.N % c != 0 || (H && BMN && c < 64)) continue;
    bn = c;
    if ((s.N / c) * n_tm * nz >= want) break;
  }
  switch (bn) {
    case 256: return tc_launch<256, AMN, BMN, H>(s, A, B, epi, st);
    case 128: return tc_launch<128, AMN, BMN, H>(s, A, B, epi, st);
    case 64: return tc_launch<64, AMN, BMN, H>(s, A, B, epi, st);
    case 32:
      if constexpr (!(H && BMN)) return tc_launch<32, AMN, BMN, H>(s, A, B, epi, st);
      break;
  }
  set_error("tc_gemm: unsupported N");
  return EDPC_ERR_INVALID;
}

}  // namespace edpc
