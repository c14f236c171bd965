// EDPC context: device-resident model, lane matrix, coders and the per-step
// schedule (predict -> quantize -> code -> backward -> Adam) behind the C ABI.
//
// Reference mapping: EdpcModel (pkg/src/edpc/model.py:184-300) and the
// compress/decompress loops (pipeline.py:109-298).  Layout, roofline and the
// determinism rules are in DESIGN.md.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <algorithm>
#include <initializer_list>
#include <type_traits>
#include <cmath>
#include <string>
#include <mutex>
#include <vector>

#include <dlfcn.h>
#include <nccl.h>

#include "common.cuh"
#include "gemm_simt.cuh"
#include "kernels.cuh"
#include "lte.cuh"
#include "tc_gemm.cuh"
#include "mbrb_fused.cuh"
#include "wgrad_adam.cuh"

namespace edpc {

// NCCL is resolved at run time (dlopen of whatever libnccl.so.2 the process
// already has -- e.g. torch's -- or the system one), only when a context joins
// a communicator, so the library never drags an NCCL into processes that do
// not use multi-GPU and never conflicts with torch's bundled NCCL.
struct NcclApi {
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t,
                       cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};

static NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.getUniqueId = (decltype(api.getUniqueId))dlsym(h, "ncclGetUniqueId");
      api.commInitRank = (decltype(api.commInitRank))dlsym(h, "ncclCommInitRank");
      api.allGather = (decltype(api.allGather))dlsym(h, "ncclAllGather");
      api.send = (decltype(api.send))dlsym(h, "ncclSend");
      api.recv = (decltype(api.recv))dlsym(h, "ncclRecv");
      api.groupStart = (decltype(api.groupStart))dlsym(h, "ncclGroupStart");
      api.groupEnd = (decltype(api.groupEnd))dlsym(h, "ncclGroupEnd");
      api.commDestroy = (decltype(api.commDestroy))dlsym(h, "ncclCommDestroy");
      api.getErrorString = (decltype(api.getErrorString))dlsym(h, "ncclGetErrorString");
      api.ok = api.getUniqueId && api.commInitRank && api.allGather && api.send && api.recv &&
               api.groupStart && api.groupEnd && api.commDestroy && api.getErrorString;
    }
  }
  return api;
}


struct MbrbOffs {
  int64_t ln_g, ln_b, w0, b0, wstride, out_w, out_b;
  int H;
};

// Offsets in the *shared* flat layout = the reference parameters() order with
// lte.lane_mats taken out (the per-lane FDM lives in its own buffers).
struct Layout {
  int T, DE, F, FP, HL, HG, K, B;
  int64_t emb, down_w, down_b, up_w, up_b, head_w, head_b;
  MbrbOffs loc, glo;
  int64_t n_shared, ref_lane_mats, n_ref, fdm;

  void build(const edpc_config& c) {
    T = c.context_len;
    DE = c.embed_dim;
    F = T * DE;
    FP = F / c.lte_ratio;
    HL = c.hidden_local;
    HG = c.hidden_global;
    K = c.branches;
    B = c.lanes;
    fdm = (int64_t)FP * FP;
    int64_t o = 0;
    emb = o;
    o += 256 * (int64_t)DE;
    auto mbrb = [&](MbrbOffs& m, int H) {
      m.H = H;
      m.ln_g = o;
      o += F;
      m.ln_b = o;
      o += F;
      m.w0 = o;
      m.b0 = o + (int64_t)F * H;
      m.wstride = (int64_t)F * H + H;
      o += K * m.wstride;
      m.out_w = o;
      o += (int64_t)H * F;
      m.out_b = o;
      o += F;
    };
    mbrb(loc, HL);
    down_w = o;
    o += (int64_t)F * FP;
    down_b = o;
    o += FP;
    ref_lane_mats = o;  // lane_mats sit here in the reference order
    up_w = o;
    o += (int64_t)FP * F;
    up_b = o;
    o += F;
    mbrb(glo, HG);
    head_w = o;
    o += (int64_t)F * 256;
    head_b = o;
    o += 256;
    n_shared = o;
    n_ref = o + (int64_t)B * fdm;
  }
};

// Per-region CUDA-event timing (bench.py's live roofline) and launch count.
enum ProfRegion {
  kRegGemm = 0, kRegFdmFwd, kRegFdmBwd, kRegAdam, kRegSoftmax, kRegEncode, kRegDecode,
  kRegColsum, kRegElem, kRegEmbed, kNumRegions
};

struct Prof {
  bool on = false;
  int64_t launches = 0;
  double ms[kNumRegions] = {};
  int64_t n[kNumRegions] = {};
  std::vector<cudaEvent_t> pool;
  struct Pair {
    cudaEvent_t a, b;
    int r;
  };
  std::vector<Pair> pending;
  cudaEvent_t open[kNumRegions] = {};

  static void chk(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fprintf(stderr, "[edpc prof] %s: %s\n", what, cudaGetErrorString(e));
  }
  cudaEvent_t get() {
    if (pool.empty()) {
      cudaEvent_t e = nullptr;
      chk(cudaEventCreate(&e), "cudaEventCreate");
      return e;
    }
    cudaEvent_t e = pool.back();
    pool.pop_back();
    return e;
  }
  void begin(int r, cudaStream_t s) {
    ++launches;
    if (!on) return;
    open[r] = get();
    chk(cudaEventRecord(open[r], s), "record(begin)");
  }
  void end(int r, cudaStream_t s) {
    if (!on || !open[r]) return;
    cudaEvent_t b = get();
    chk(cudaEventRecord(b, s), "record(end)");
    pending.push_back({open[r], b, r});
    open[r] = nullptr;
  }
  void flush() {
    for (auto& p : pending) {
      chk(cudaEventSynchronize(p.b), "sync");
      float t = 0.f;
      chk(cudaEventElapsedTime(&t, p.a, p.b), "elapsed");
      ms[p.r] += t;
      n[p.r] += 1;
      pool.push_back(p.a);
      pool.push_back(p.b);
    }
    pending.clear();
  }
  void reset() {
    flush();
    launches = 0;
    for (int r = 0; r < kNumRegions; ++r) ms[r] = 0, n[r] = 0;
  }
  void release() {
    for (auto& p : pending) {
      chk(cudaEventDestroy(p.a), "destroy");
      chk(cudaEventDestroy(p.b), "destroy");
    }
    pending.clear();
    for (auto e : pool) chk(cudaEventDestroy(e), "destroy");
    pool.clear();
  }
};

}  // namespace edpc

using namespace edpc;

struct edpc_ctx {
  Prof prof;
  edpc_config cfg;
  Layout lay;
  int device = 0;
  int Bl = 0, lane0 = 0, S = 0, Sl = 0, spl = 0, seg0 = 0;
  int64_t n = 0, L = 0;
  int g_first = 0, g_count = 0;  // local lane groups
  bool use_tc = false;
  // fp16 GEMM path for the MBRB branch / out-projection GEMMs (see ctx_create)
  bool h16 = false;
  bool lte_fwd = false;  // fused LTE forward kernel (numerics bit 2)
  // tf32 GEMM operands rounded to nearest (numerics bit 3): weights from the
  // tf32-rounded shadow Wt, activations stored rounded by their producers
  bool rt = false;
  float* Wt = nullptr;
  // weight gradient + lane-group tree + Adam fused (wgrad_adam.cuh): one
  // context holding all 8 lane groups on the tensor-core path
  bool wfuse = false;
  // weight gradients as two subtree partials (groups 0-3 -> slot 0, 4-7 ->
  // slot 4) instead of 8 per-group partials; Adam's top tree level over them
  bool wsub = false;
  bool keep_grads = false;  // debug: fused kernels also write the reduced gradient to Gp slot 0
  int64_t arr = 0;          // W -> M -> V distance (one allocation)
  int gs_log2 = 0;                                  // gradient scale 2^gs_log2 (k_dlogits)
  __half* Wh = nullptr;                             // fp16 shadow of the shared weights
  __half *guph_l = nullptr, *guph_g = nullptr;      // fp16 copies of g_up per MBRB
  cudaStream_t st = nullptr, st_enc = nullptr;
  cudaStream_t st_aux = nullptr;  // weight-gradient GEMMs run here, joined before Adam
  cudaStream_t st_h2d = nullptr;  // streaming ingest of input columns (edpc_set_input_columns)
  cudaEvent_t ev_h2d = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev = nullptr;
  cudaEvent_t t0 = nullptr, t1 = nullptr, tj = nullptr;
  cudaGraphExec_t graph[2] = {nullptr, nullptr};
  ncclComm_t comm = nullptr;  // multi-GPU: slice exchange of subtree sums + weight all-gather
  int nranks = 1, rank = 0;
  AdamConsts adam{};

  std::vector<void*> allocs;
  float *W = nullptr, *M = nullptr, *V = nullptr, *Gp = nullptr;
  float *U = nullptr, *Um = nullptr, *Uv = nullptr;
  cudaAccessPolicyWindow l2win{};  // persisting-L2 window over U (num_bytes 0: none)
  uint8_t* mat = nullptr;
  uint8_t* scratch = nullptr;  // [Bl][T+1] for the predict/train_step seam
  int64_t *d_i = nullptr, *d_t = nullptr;
  // activations
  float *x_emb, *l_xhat, *l_rstd, *l_x0, *l_H, *l_ff, *x_local;
  float *down, *mixed, *x_lte;
  float *g_xhat, *g_rstd, *g_x0, *g_H, *g_ff, *x_global;
  float *logits, *probs, *nll;
  // backward temporaries
  float *gl, *gx0, *gmix, *gdown, *emb_sub;
  float *g_head, *g_lte, *g_loc, *g_emb;  // dL/d(x_global), d(x_lte), d(x_local), d(x_emb)
  float *GH_g, *GH_l;                     // branch-output gradients per MBRB
  float* ws = nullptr;  // split-K workspace [kSplitK][Bl][<=256]
  float* ln_scratch = nullptr;  // LN-gradient chunk sums
  unsigned* ln_tickets = nullptr;
  int *chunk_tab = nullptr, *grp_chunks = nullptr;
  int n_chunks = 0;
  // coder
  uint32_t* intervals = nullptr;
  uint16_t* cdf16 = nullptr;
  int64_t *enc_state = nullptr, *dec_state = nullptr;
  uint32_t* enc_words = nullptr;
  int64_t enc_cap_words = 0;
  uint8_t* payload = nullptr;
  uint8_t* packed = nullptr;  // assembled payload area (compress_finish)
  int64_t packed_bytes = 0;
  int64_t *pay_off = nullptr, *bit_len = nullptr;
  int* dec_err = nullptr;
  // host bookkeeping
  int64_t enc_upto = 0;   // intervals columns [0, enc_upto) handed to the encoder
  int64_t cols_done = 0;  // lane columns whose intervals have been produced
  bool finished = false, have_input = false, have_payload = false, have_cache = false;
  int64_t version = 0;   // model updates done (seam)
  int64_t seam_t = 0;

  ~edpc_ctx() {
    if (st) cudaStreamSynchronize(st);
    if (st_enc) cudaStreamSynchronize(st_enc);
    if (st_aux) cudaStreamSynchronize(st_aux);
    if (st_h2d) cudaStreamSynchronize(st_h2d);
    prof.flush();
    prof.release();
    for (auto& g : graph)
      if (g) cudaGraphExecDestroy(g);
    if (l2win.num_bytes) cudaCtxResetPersistingL2Cache();
    if (comm) nccl().commDestroy(comm);
    // back to the device's stream-ordered pool (kept resident: the next
    // context's allocations reuse it instead of cudaMalloc/cudaFree round trips)
    for (void* p : allocs) cudaFreeAsync(p, st);
    if (ev) cudaEventDestroy(ev);
    if (t0) cudaEventDestroy(t0);
    if (t1) cudaEventDestroy(t1);
    if (tj) cudaEventDestroy(tj);
    if (st) cudaStreamDestroy(st);
    if (st_enc) cudaStreamDestroy(st_enc);
    if (st_aux) cudaStreamDestroy(st_aux);
    if (st_h2d) cudaStreamDestroy(st_h2d);
    if (ev_h2d) cudaEventDestroy(ev_h2d);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
  }

  template <typename T>
  int alloc(T** p, int64_t count) {
    size_t bytes = (size_t)std::max<int64_t>(count, 1) * sizeof(T);
    bytes = (bytes + 255) & ~(size_t)255;
    void* q = nullptr;
    // stream-ordered pool allocation, complete before any other stream uses it
    cudaError_t e = cudaMallocAsync(&q, bytes, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
      set_error("cudaMallocAsync(" + std::to_string(bytes) + "): " + cudaGetErrorString(e));
      return EDPC_ERR_NOMEM;
    }
    allocs.push_back(q);
    *p = reinterpret_cast<T*>(q);
    return EDPC_OK;
  }

  int step_off = 0;  // model steps since d_i / d_t were last advanced (inside a graph capture)
  StepIdx si() const { return StepIdx{d_i, d_t, step_off}; }
  ByteCols lanes_src() const { return ByteCols{mat, L}; }
  ByteCols seam_src() const { return ByteCols{scratch, (int64_t)lay.T + 1}; }
};

namespace edpc {

constexpr int kTf32MinLanes = 1024;
// numerics flags (edpc_ctx_numerics / edpc_ctx_create_ex, container header)
constexpr int kNumTc = 1, kNumF16 = 2, kNumLteFused = 4, kNumRndTf32 = 8, kNumericsMask = 15;

// B operand of a tf32 GEMM: the tf32-rounded weight shadow when the context
// rounds tf32 operands (numerics bit 3), else the fp32 master weights
static const float* wt(const edpc_ctx* c) { return c->rt ? c->Wt : c->W; }

constexpr int kFdmWarps = 2;  // warps per block of the per-lane FDM kernels

static bool sync_debug() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("EDPC_SYNC_DEBUG");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

// Brackets one kernel launch: launch count, optional CUDA-event timing, and
// (EDPC_SYNC_DEBUG=1) a synchronous error check naming the region.
struct Scope {
  edpc_ctx* c;
  int r;
  cudaStream_t s;
  const char* where;
  Scope(edpc_ctx* c_, int r_, cudaStream_t s_, const char* w = "")
      : c(c_), r(r_), s(s_), where(w) {
    c->prof.begin(r, s);
  }
  ~Scope() {
    c->prof.end(r, s);
    if (sync_debug()) {
      cudaError_t e = cudaStreamSynchronize(s);
      if (e == cudaSuccess) e = cudaGetLastError();
      if (e != cudaSuccess) {
        fprintf(stderr, "[edpc debug] region %d (%s) launch #%lld failed: %s\n", r, where,
                (long long)c->prof.launches, cudaGetErrorString(e));
        abort();
      }
    }
  }
};

static int check_cfg(const edpc_config* c) {
  EDPC_CHECK_ARG(c, "null config");
  EDPC_CHECK_ARG(c->context_len >= 1, "context_len must be >= 1");
  EDPC_CHECK_ARG(c->embed_dim >= 1, "embed_dim must be >= 1");
  EDPC_CHECK_ARG(c->branches >= 1, "branches must be >= 1");
  EDPC_CHECK_ARG(c->branches <= kMaxBranches, "branches > 8 unsupported");
  EDPC_CHECK_ARG(c->lanes >= 1, "lanes must be >= 1");
  EDPC_CHECK_ARG(c->hidden_local >= 1 && c->hidden_global >= 1, "hidden dims must be >= 1");
  int64_t f = (int64_t)c->context_len * c->embed_dim;
  EDPC_CHECK_ARG(c->lte_ratio >= 1 && f % c->lte_ratio == 0,
                 "lte_ratio must divide context_len * embed_dim");
  EDPC_CHECK_ARG(c->context_len <= 4096, "context_len > 4096 unsupported");
  return EDPC_OK;
}

// ------------------------------------------------------------ GEMM dispatch

static bool al16(const void* p) { return ((uintptr_t)p & 15) == 0; }

// tcgen05 path eligibility: shapes that tile cleanly and 16-byte aligned
// operands / strides (TMA).  The choice depends only on the config and the
// buffer layout, so compress and decompress always take the same path.
static bool tc_ok_m(edpc_ctx* c, int bit, int N, int Kchunk,
                    std::initializer_list<const void*> ptrs,
                    std::initializer_list<int64_t> strides);

static bool tc_ok(edpc_ctx* c, int N, int Kchunk, std::initializer_list<const void*> ptrs,
                  std::initializer_list<int64_t> strides) {
  if (!c->use_tc || !tc_shape_ok(N, Kchunk)) return false;
  for (const void* p : ptrs)
    if (!al16(p)) return false;
  for (int64_t s : strides)
    if (s % 4) return false;
  return true;
}

static bool tc_ok_m(edpc_ctx* c, int bit, int N, int Kchunk,
                    std::initializer_list<const void*> ptrs,
                    std::initializer_list<int64_t> strides) {
  (void)bit;
  return tc_ok(c, N, Kchunk, ptrs, strides);
}

static cudaError_t as_cuda(int st) { return st == EDPC_OK ? cudaSuccess : cudaErrorUnknown; }

// Skinny-N GEMMs (N <= 256, long K) give only Bl/128 output tiles; split K
// kSplitK ways so the grid covers the SMs, then reduce in a fixed order.
constexpr int kSplitK = 4;
static bool use_split(int N, int64_t Ktot, int Kd) {
  return N <= 256 && N % 4 == 0 && Ktot >= 1024 && Kd % (kSplitK * kTcBK) == 0;
}

static cudaError_t splitk_reduce(edpc_ctx* c, int N, const float* bias, const float* resid,
                                 float* out, int rt) {
  const int64_t plane = (int64_t)c->Bl * N;
  Scope sc(c, kRegElem, c->st);
  pdl_launch(k_splitk_reduce, (unsigned)cdiv(plane / 4, 256), 256, 0, c->st, c->ws, kSplitK, plane, N, bias,
                                                                    resid, out, rt);
  return cudaGetLastError();
}

// one split-K GEMM into out (+ bias) (+ resid): EpiSplit partials + k_splitk_reduce.
// (Reducing inside the GEMM -- the last CTA of a tile, or all of a tile's CTAs
// after a wait -- measured slower at C2: 7.35 / 7.74 vs 8.14 MB/s; CTAs that
// stay resident to reduce hold SMs the side-stream weight-gradient GEMMs need.)
template <bool AMN, bool BMN, bool H = false>
static cudaError_t split_gemm(edpc_ctx* c, const TcShape& s, const TcOperand& a, const TcOperand& b,
                              const float* bias, const float* resid, float* out, int rt = 0) {
  const int N = s.N;
  const int64_t plane = (int64_t)c->Bl * N;
  {
    Scope sc(c, kRegGemm, c->st);
    int st = tc_gemm<AMN, BMN, H>(s, a, b, EpiSplit{c->ws, N, plane}, c->st);
    if (st != EDPC_OK) return cudaErrorUnknown;
  }
  return splitk_reduce(c, N, bias, resid, out, rt);
}

// out[Bl][N] = A[Bl][Kd] . W[Kd][N] (+ bias) over nzb batches (weights at
// w + z*sW, bias at bias + z*sW, out at out + z*sOut)
static cudaError_t fwd_linear(edpc_ctx* c, const float* A, int lda, int Kd, const float* w,
                              int N, int nzb, int64_t sW, float* out, int64_t sOut,
                              const float* bias, const float* resid, int M) {
  if (tc_ok_m(c, 0, N, Kd, {A, w, out, bias, resid ? resid : out}, {lda, N, sW, sOut})) {
    TcOperand a{A, lda, 0, 1}, b{w, N, sW, nzb};
    if (nzb == 1 && M == c->Bl && use_split(N, Kd, Kd)) {
      TcShape s{M, N, Kd, 1, 1, kBatchNone, kBatchNone, 2, kSplitK, 0, 0, 0};
      return split_gemm<false, true>(c, s, a, b, bias, resid, out, resid ? c->rt : 0);
    }
    Scope sc(c, kRegGemm, c->st);
    TcShape s{M, N, Kd, nzb, 1, kBatchNone, nzb > 1 ? kBatchZ : kBatchNone, 0, 1, 0, 0, 0};
    if (resid)
      return as_cuda(tc_gemm<false, true>(s, a, b, EpiBiasResid{out, N, bias, resid, N, c->rt}, c->st));
    return as_cuda(tc_gemm<false, true>(s, a, b, EpiBias{out, N, sOut, bias, sW}, c->st));
  }
  Scope sc(c, kRegGemm, c->st);
  GemmShape g{};
  g.M = M;
  g.N = N;
  g.K = Kd;
  g.A = A;
  g.lda = lda;
  g.B = w;
  g.ldb = N;
  g.sB = sW;
  g.nzb = nzb;
  g.nsum = 1;
  if (resid) return gemm_simt<false, false>(g, EpiBiasResid{out, N, bias, resid, N, c->rt}, c->st);
  return gemm_simt<false, false>(g, EpiBias{out, N, sOut, bias, sW}, c->st);
}

static cudaError_t colsum(edpc_ctx* c, const float* src, int N, int nz, int64_t sz,
                          const float* mul, int64_t off, int64_t sOff, cudaStream_t st = nullptr);

// weight-gradient partials: Gp[g][off + z*sOff + m*N + n] = sum over group
// g's lanes of X[b][m] * G[z][b][n], and (bias_off >= 0) the bias partials
// Gp[g][bias_off + z*sOff + n] = sum over the group's lanes of G[z][b][n] --
// on the tcgen05 path those come from the GEMM's own B tiles in shared memory.
static bool aux_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("EDPC_AUX_STREAM");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

// work of the weight-gradient stream (joined back before the exchange / Adam)
static cudaStream_t wst(edpc_ctx* c) { return aux_enabled() ? c->st_aux : c->st; }

static cudaError_t fork_aux(edpc_ctx* c) {
  if (!aux_enabled()) return cudaSuccess;
  cudaError_t e = cudaEventRecord(c->ev_fork, c->st);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(c->st_aux, c->ev_fork, 0);
  return e;
}

static cudaError_t join_aux(edpc_ctx* c) {
  if (!aux_enabled()) return cudaSuccess;
  cudaError_t e = cudaEventRecord(c->ev_join, c->st_aux);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(c->st, c->ev_join, 0);
  return e;
}

static WgAdamArgs wgrad_adam_args(edpc_ctx* c, int64_t off, int64_t sOff, int64_t bias_off, int N,
                                  bool half) {
  WgAdamArgs a{};
  a.B_global = c->lay.B;
  a.lane0 = c->lane0;
  a.bias_off = bias_off;
  a.bias_zstride = sOff;
  a.W = c->W;
  a.arr = c->arr;
  a.Wh = half ? c->Wh : nullptr;
  a.Wt = (!half && c->rt) ? c->Wt : nullptr;
  a.si = c->si();
  a.ac = c->adam;
  a.b1d = c->cfg.beta1;
  a.b2d = c->cfg.beta2;
  a.ginv = ldexpf(1.0f, -c->gs_log2);
  a.keep = c->keep_grads ? c->Gp : nullptr;
  a.keep_off = off;
  a.keep_ld = N;
  a.keep_zs = sOff;
  return a;
}

template <bool H>
static cudaError_t wgrad_sub(edpc_ctx* c, const void* X, int Mw, const void* G, int N, int nzb,
                             int64_t sG, int64_t off, int64_t sOff, int64_t bias_off) {
  Scope sc(c, kRegGemm, wst(c));
  const int B = c->lay.B;
  const int64_t P = c->lay.n_shared;
  if (N % 128 == 0)
    return as_cuda(wgrad_subtree_launch<H, 128>(X, Mw, G, N, nzb, sG, B, c->lane0, c->Gp, P, off,
                                                sOff, bias_off, wst(c)));
  return as_cuda(wgrad_subtree_launch<H, 64>(X, Mw, G, N, nzb, sG, B, c->lane0, c->Gp, P, off, sOff,
                                             bias_off, wst(c)));
}

static cudaError_t wgrad(edpc_ctx* c, const float* X, int Mw, const float* G, int N, int nzb,
                         int64_t sG, int64_t off, int64_t sOff, int64_t bias_off) {
  if (c->wsub) return wgrad_sub<false>(c, X, Mw, G, N, nzb, sG, off, sOff, bias_off);
  if (c->wfuse) {  // gradient + tree + Adam in one kernel (no partials, no Adam launch)
    Scope sc(c, kRegGemm, wst(c));
    return as_cuda(wgrad_adam_launch<false>(X, Mw, G, N, nzb, sG,
                                            wgrad_adam_args(c, off, sOff, bias_off, N, false), off,
                                            sOff, wst(c)));
  }
  EpiPartial e{c->Gp, c->lay.n_shared, off, sOff, N, c->g_first};
  cudaStream_t ws = wst(c);
  const int glanes = c->lay.B / kNumGroups;
  if (c->lay.B % kNumGroups == 0 && glanes % kTcBK == 0 &&
      tc_ok_m(c, 3, N, glanes, {X, G, c->Gp + off}, {Mw, N, sG, sOff, c->lay.n_shared})) {
    Scope sc(c, kRegGemm, ws);
    TcShape s{Mw, N, c->Bl, nzb, 1, kBatchNone, nzb > 1 ? kBatchZ : kBatchNone, 1,
              c->g_count, c->g_first, c->lay.B, c->lane0};
    if (bias_off >= 0) {
      s.bias_part = c->Gp;
      s.bias_gstride = c->lay.n_shared;
      s.bias_off = bias_off;
      s.bias_zstride = sOff;
    }
    TcOperand a{X, Mw, 0, 1}, b{G, N, sG, nzb};
    return as_cuda(tc_gemm<true, true>(s, a, b, e, ws));
  }
  {
    Scope sc(c, kRegGemm, ws);
    GemmShape g{};
    g.M = Mw;
    g.N = N;
    g.K = c->Bl;
    g.A = X;
    g.lda = Mw;
    g.B = G;
    g.ldb = N;
    g.sB = sG;
    g.nzb = nzb;
    g.nsum = 1;
    g.ngroups = c->g_count;
    g.g0 = c->g_first;
    g.B_global = c->lay.B;
    g.lane0 = c->lane0;
    cudaError_t r = gemm_simt<true, false>(g, e, ws);
    if (r != cudaSuccess) return r;
  }
  if (bias_off >= 0) return colsum(c, G, N, nzb, sG, nullptr, bias_off, sOff, ws);
  return cudaSuccess;
}

// bias-gradient partials (column sums per lane group)
static cudaError_t colsum(edpc_ctx* c, const float* src, int N, int nz, int64_t sz,
                          const float* mul, int64_t off, int64_t sOff, cudaStream_t st) {
  if (c->g_count == 0) return cudaSuccess;
  if (!st) st = c->st;
  const int vec = (N % 4 == 0 && sz % 4 == 0 && al16(src) && (!mul || al16(mul))) ? 1 : 0;
  dim3 grid((unsigned)cdiv(N, 128), (unsigned)nz, (unsigned)c->g_count);
  Scope sc(c, kRegColsum, st);
  pdl_launch(k_colsum_groups, grid, 256, 0, st, src, N, sz, mul, N, c->Gp, c->lay.n_shared, off, sOff,
                                           c->g_first, c->lay.B, c->lane0, vec);
  return cudaGetLastError();
}

// dgrad: out[Bl][N] = sum_s G_s[Bl][Kd] . W_s^T where W_s is [N][Kd] row-major
template <class Epi>
static cudaError_t dgrad(edpc_ctx* c, const float* G, int Kd, int nsum, int64_t sG_sum,
                         const float* w, int64_t sW_sum, int N, const Epi& epi) {
  if (tc_ok_m(c, 2, N, Kd, {G, w}, {Kd, sG_sum, sW_sum})) {
    TcOperand a{G, Kd, sG_sum, nsum}, b{w, Kd, sW_sum, nsum};
    if constexpr (std::is_same<Epi, EpiStore>::value) {
      if (epi.ldc == N && use_split(N, (int64_t)Kd * nsum, Kd)) {
        TcShape s{c->Bl, N, Kd, 1, nsum, nsum > 1 ? kBatchSum : kBatchNone,
                  nsum > 1 ? kBatchSum : kBatchNone, 2, kSplitK, 0, 0, 0};
        return split_gemm<false, false>(c, s, a, b, nullptr, nullptr, epi.C);
      }
    }
    Scope sc(c, kRegGemm, c->st);
    TcShape s{c->Bl, N, Kd, 1, nsum, nsum > 1 ? kBatchSum : kBatchNone,
              nsum > 1 ? kBatchSum : kBatchNone, 0, 1, 0, 0, 0};
    return as_cuda(tc_gemm<false, false>(s, a, b, epi, c->st));
  }
  Scope sc(c, kRegGemm, c->st);
  GemmShape g{};
  g.M = c->Bl;
  g.N = N;
  g.K = Kd;
  g.A = G;
  g.lda = Kd;
  g.sA_sum = sG_sum;
  g.B = w;
  g.ldb = Kd;
  g.sB_sum = sW_sum;
  g.nzb = 1;
  g.nsum = nsum;
  return gemm_simt<false, true>(g, epi, c->st);
}

// ---------------------------------------------------- fp16 GEMM path
//
// The MBRB branch and out-projection GEMMs (>90% of the step's FLOPs) take
// fp16 operands (kind::f16: 2x the tf32 MMA rate, half the operand bytes):
// x0, ff, D_z and g_H are stored as fp16 by the kernels that produce them,
// the weights come from an fp16 shadow refreshed by Adam, g_up gets an fp16
// copy.  fp16 has tf32's 10-bit mantissa (rounded, not truncated); range is
// handled by the power-of-two gradient scale (k_dlogits).

static cudaError_t fwd_linear_h(edpc_ctx* c, const __half* A, int Kd, const __half* w, int N,
                                float* out, const float* bias, const float* resid) {
  const int M = c->Bl;
  TcOperand a{A, Kd, 0, 1}, b{w, N, 0, 1};
  if (N <= 256 && N % 4 == 0 && Kd >= 1024 && Kd % (kSplitK * tc_bk<true>()) == 0) {
    TcShape s{M, N, Kd, 1, 1, kBatchNone, kBatchNone, 2, kSplitK, 0, 0, 0};
    return split_gemm<false, true, true>(c, s, a, b, bias, resid, out, resid ? c->rt : 0);
  }
  Scope sc(c, kRegGemm, c->st);
  TcShape s{M, N, Kd, 1, 1, kBatchNone, kBatchNone, 0, 1, 0, 0, 0};
  if (resid)
    return as_cuda(
        tc_gemm<false, true, true>(s, a, b, EpiBiasResid{out, N, bias, resid, N, c->rt}, c->st));
  return as_cuda(tc_gemm<false, true, true>(s, a, b, EpiBias{out, N, 0, bias, 0}, c->st));
}

// out[Bl][N] = sum_s G_s[Bl][Kd] . W_s^T, W_s fp16 [N][Kd]
static cudaError_t dgrad_h(edpc_ctx* c, const __half* G, int Kd, int nsum, int64_t sG_sum,
                           const __half* w, int64_t sW_sum, int N, float* out) {
  TcOperand a{G, Kd, sG_sum, nsum}, b{w, Kd, sW_sum, nsum};
  const TcBatch bt = nsum > 1 ? kBatchSum : kBatchNone;
  if (N <= 256 && N % 4 == 0 && (int64_t)Kd * nsum >= 1024 &&
      Kd % (kSplitK * tc_bk<true>()) == 0) {
    TcShape s{c->Bl, N, Kd, 1, nsum, bt, bt, 2, kSplitK, 0, 0, 0};
    return split_gemm<false, false, true>(c, s, a, b, nullptr, nullptr, out);
  }
  Scope sc(c, kRegGemm, c->st);
  TcShape s{c->Bl, N, Kd, 1, nsum, bt, bt, 0, 1, 0, 0, 0};
  return as_cuda(tc_gemm<false, false, true>(s, a, b, EpiStore{out, N}, c->st));
}

// weight-gradient partials from fp16 X [lanes][Mw] and G [nzb][lanes][N]
// (both MN-major operands: K = lanes, split into the lane groups)
// and (bias_off >= 0) the bias partials = column sums of G over the group's
// lanes, by the GEMM's bias warps from its own fp16 B tiles in shared memory
static cudaError_t wgrad_h(edpc_ctx* c, const __half* X, int Mw, const __half* G, int N, int nzb,
                           int64_t sG, int64_t off, int64_t sOff, int64_t bias_off) {
  if (c->wsub) return wgrad_sub<true>(c, X, Mw, G, N, nzb, sG, off, sOff, bias_off);
  if (c->wfuse) {
    Scope sc(c, kRegGemm, wst(c));
    return as_cuda(wgrad_adam_launch<true>(X, Mw, G, N, nzb, sG,
                                           wgrad_adam_args(c, off, sOff, bias_off, N, true), off,
                                           sOff, wst(c)));
  }
  EpiPartial e{c->Gp, c->lay.n_shared, off, sOff, N, c->g_first};
  cudaStream_t ws = wst(c);
  Scope sc(c, kRegGemm, ws);
  TcShape s{Mw, N, c->Bl, nzb, 1, kBatchNone, nzb > 1 ? kBatchZ : kBatchNone, 1,
            c->g_count, c->g_first, c->lay.B, c->lane0};
  if (bias_off >= 0) {
    s.bias_part = c->Gp;
    s.bias_gstride = c->lay.n_shared;
    s.bias_off = bias_off;
    s.bias_zstride = sOff;
  }
  TcOperand a{X, Mw, 0, 1}, b{G, N, sG, nzb};
  return as_cuda(tc_gemm<true, true, true>(s, a, b, e, ws));
}


#define CK(expr)                                                        \
  do {                                                                  \
    cudaError_t _e = (expr);                                            \
    if (_e != cudaSuccess) {                                            \
      set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));    \
      return EDPC_ERR_CUDA;                                             \
    }                                                                   \
  } while (0)

// --------------------------------------------------------------- forward

// The fused MBRB forward (mbrb_fused.cuh) is bit-identical to the two-GEMM
// path; EDPC_MBRB_FUSED=0 selects the latter for A/B timing.
static bool mbrb_fused_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("EDPC_MBRB_FUSED");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

struct MbrbBufs {
  float *x, *xhat, *rstd, *x0, *H, *ff, *out;
};

static int mbrb_forward(edpc_ctx* c, const MbrbOffs& o, const MbrbBufs& b, bool gather,
                        ByteCols src, bool ln_done = false) {
  const Layout& L = c->lay;
  const int Bl = c->Bl, F = L.F, H = o.H;
  dim3 g8((unsigned)cdiv(Bl, 8));
  if (!ln_done) {
    Scope sc_ln(c, kRegElem, c->st);
    __half* x0h = c->h16 ? reinterpret_cast<__half*>(b.x0) : nullptr;
    if (gather)
      pdl_launch(k_embed_ln<true>, g8, 256, 0, c->st, src, c->si(), L.T, c->W + L.emb, L.DE, F, Bl, b.x,
                                              c->W + o.ln_g, c->W + o.ln_b, b.xhat, b.rstd, b.x0,
                                              x0h, (int)c->rt);
    else
      pdl_launch(k_embed_ln<false>, g8, 256, 0, c->st, src, c->si(), L.T, c->W + L.emb, L.DE, F, Bl, b.x,
                                               c->W + o.ln_g, c->W + o.ln_b, b.xhat, b.rstd, b.x0,
                                               x0h, (int)c->rt);
    CK(cudaGetLastError());
  }
  const int64_t plane = (int64_t)Bl * H;
  if (c->h16) {  // fp16 operands; x0, ff and D_z live in their buffers as fp16
    __half* x0h = reinterpret_cast<__half*>(b.x0);
    __half* ffh = reinterpret_cast<__half*>(b.ff);
    __half* Dh = reinterpret_cast<__half*>(b.H);
    if (mbrb_fused_enabled() && mbrb_fused_ok(F, H, L.K)) {
      // branch GEMMs + product/GeLU + out-projection in one kernel (hidden
      // tile on chip; the fixed-order split reduction with bias and residual
      // over DSMEM in the same kernel) -- bit-identical to the two-GEMM path
      Scope sc(c, kRegGemm, c->st);
      return mbrb_fwd_fused(x0h, c->Wh + o.w0, o.wstride, c->Wh + o.out_w, c->W + o.b0, Bl, H, ffh,
                            Dh, c->W + o.out_b, b.x, b.out, (int)c->rt, c->st);
    }
    {
      Scope sc(c, kRegGemm, c->st);
      TcShape s{Bl, H, F, 2, 1, kBatchNone, kBatchZ, 0, 1, 0, 0, 0};
      TcOperand a{x0h, F, 0, 1}, bw{c->Wh + o.w0, H, o.wstride, 2};
      const int st = tc_launch_zin<128, 2, true, true>(
          s, a, bw, EpiBranchActH<2>{Dh, ffh, c->W + o.b0, o.wstride, H, plane}, c->st);
      if (st != EDPC_OK) return st;
    }
    CK(fwd_linear_h(c, ffh, H, c->Wh + o.out_w, F, b.out, c->W + o.out_b, b.x));
    return EDPC_OK;
  }
  // branch GEMMs with the product + GeLU fused into the epilogue when all
  // branches of a tile fit one CTA's TMEM (k = 2, 3); else GEMM + k_mbrb_act
  if ((L.K == 2 || L.K == 3) && H % 128 == 0 &&
      tc_ok_m(c, 1, H, F, {b.x0, wt(c) + o.w0, b.H, b.ff, c->W + o.b0}, {F, H, o.wstride, plane})) {
    Scope sc(c, kRegGemm, c->st);
    TcShape s{Bl, H, F, L.K, 1, kBatchNone, kBatchZ, 0, 1, 0, 0, 0};
    TcOperand a{b.x0, F, 0, 1}, bw{wt(c) + o.w0, H, o.wstride, L.K};
    const int rt = c->rt;
    const int st =
        L.K == 2 ? tc_launch_zin<128, 2, true>(
                       s, a, bw, EpiBranchAct<2>{b.H, b.ff, c->W + o.b0, o.wstride, H, plane, rt},
                       c->st)
                 : tc_launch_zin<64, 3, true>(
                       s, a, bw, EpiBranchAct<3>{b.H, b.ff, c->W + o.b0, o.wstride, H, plane, rt},
                       c->st);
    if (st != EDPC_OK) return st;
  } else {
    CK(fwd_linear(c, b.x0, F, F, wt(c) + o.w0, H, L.K, o.wstride, b.H, plane, c->W + o.b0, nullptr,
                  Bl));
    Scope sc_(c, kRegElem, c->st);
    pdl_launch(k_mbrb_act, (unsigned)cdiv(plane, 256), 256, 0, c->st, b.H, L.K, plane, b.ff,
               (int)c->rt);
    CK(cudaGetLastError());
  }
  CK(fwd_linear(c, b.ff, H, H, wt(c) + o.out_w, F, 1, 0, b.out, 0, c->W + o.out_b, b.x, Bl));
  return EDPC_OK;
}

// Fused LTE forward (lte.cuh, k_lte_fwd): paper dims on the tcgen05 path (the
// SIMT path keeps the reference-shaped GEMM -> FDM -> GEMM sequence).  ncu:
// 24.8 us vs 39.7 us for the three launches.  Part of the numerics (mma.sync
// tf32 rounds operands to nearest, tcgen05 tf32 truncates): numerics bit 2.
static bool lte_fused(const edpc_ctx* c) { return c->lte_fwd; }

// the global MBRB's layer norm inside k_lte_fwd (bit-identical to the
// separate k_embed_ln; EDPC_LTE_LN_FUSED=0 selects the latter for A/B runs)
static bool lte_ln_fused() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("EDPC_LTE_LN_FUSED");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

static bool lte_fused_possible(const edpc_ctx* c) {
  if (!(c->use_tc && c->lay.F == lte::kF && c->lay.FP == lte::kFP)) return false;
  static signed char attr[64] = {};  // per device: 0 unset, 1 ok, -1 failed
  signed char& a = attr[c->device & 63];
  if (a == 0) {
    a = cudaFuncSetAttribute(k_lte_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)lte::kSmemBytesF) == cudaSuccess
            ? 1
            : -1;
  }
  return a == 1;
}

static int forward(edpc_ctx* c, ByteCols src) {
  const Layout& L = c->lay;
  const int Bl = c->Bl;
  MbrbBufs lb{c->x_emb, c->l_xhat, c->l_rstd, c->l_x0, c->l_H, c->l_ff, c->x_local};
  EDPC_TRY(mbrb_forward(c, L.loc, lb, true, src));
  if (lte_fused(c)) {
    Scope sc_(c, kRegFdmFwd, c->st);
    // + the global MBRB's layer norm (its k_embed_ln launch disappears)
    const bool ln = lte_ln_fused();
    pdl_launch(k_lte_fwd, (unsigned)cdiv(Bl, lte::kRows), lte::kThreads, lte::kSmemBytesF, c->st,
               c->x_local, c->W + L.down_w, c->W + L.down_b, c->U, c->W + L.up_w, c->W + L.up_b,
               c->down, c->mixed, c->x_lte, Bl, ln ? c->W + L.glo.ln_g : nullptr,
               c->W + L.glo.ln_b, c->g_xhat, c->g_rstd, c->g_x0,
               c->h16 ? reinterpret_cast<__half*>(c->g_x0) : nullptr, (int)c->rt);
    CK(cudaGetLastError());
  } else {
  CK(fwd_linear(c, c->x_local, L.F, L.F, wt(c) + L.down_w, L.FP, 1, 0, c->down, 0,
                c->W + L.down_b, nullptr, Bl));
  {
    Scope sc_(c, kRegFdmFwd, c->st);
    if (L.FP == 64 || L.FP == 128 || L.FP == 256) {
    // 2-warp blocks: 256-thread blocks left 108 SMs with two blocks and 40
    // with one (all resident at once), 86% balance; 64-thread blocks ~99%
    const int lpw = 32 / std::min(32, L.FP / 4);
    const unsigned blocks = (unsigned)cdiv(cdiv(Bl, lpw), kFdmWarps);
    if (L.FP == 64)
      pdl_launch(k_fdm_fwd_v<64>, blocks, 32 * kFdmWarps, 0, c->st, c->down, c->U, c->mixed, Bl,
                 (int)c->rt);
    else if (L.FP == 128)
      pdl_launch(k_fdm_fwd_v<128>, blocks, 32 * kFdmWarps, 0, c->st, c->down, c->U, c->mixed, Bl,
                 (int)c->rt);
    else
      pdl_launch(k_fdm_fwd_v<256>, blocks, 32 * kFdmWarps, 0, c->st, c->down, c->U, c->mixed, Bl,
                 (int)c->rt);
  } else {
    pdl_launch(k_fdm_fwd, (unsigned)cdiv(Bl, 8), 256, 0, c->st, c->down, c->U, c->mixed, L.FP, Bl,
               (int)c->rt);
  }
  }
  CK(cudaGetLastError());
  CK(fwd_linear(c, c->mixed, L.FP, L.FP, wt(c) + L.up_w, L.F, 1, 0, c->x_lte, 0, c->W + L.up_b,
                nullptr, Bl));
  }
  MbrbBufs gb{c->x_lte, c->g_xhat, c->g_rstd, c->g_x0, c->g_H, c->g_ff, c->x_global};
  EDPC_TRY(mbrb_forward(c, L.glo, gb, false, src, lte_fused(c) && lte_ln_fused()));
  CK(fwd_linear(c, c->x_global, L.F, L.F, wt(c) + L.head_w, 256, 1, 0, c->logits, 0,
                c->W + L.head_b, nullptr, Bl));
  return EDPC_OK;
}

static int softmax_quant(edpc_ctx* c, int mode, ByteCols src) {
  dim3 g8((unsigned)cdiv(c->Bl, 8));
  Scope sc(c, kRegSoftmax, c->st);
  const float Bf = (float)c->lay.B, gs = ldexpf(1.0f, c->gs_log2);
  if (mode == kProbsOnly)
    pdl_launch(k_softmax_quant<kProbsOnly>, g8, 256, 0, c->st, c->logits, c->probs, c->Bl, src,
               c->si(), c->intervals, c->cdf16, Bf, gs, nullptr);
  else if (mode == kEncode)  // also the loss gradient (backward skips k_dlogits)
    pdl_launch(k_softmax_quant<kEncode>, g8, 256, 0, c->st, c->logits, c->probs, c->Bl, src,
               c->si(), c->intervals, c->cdf16, Bf, gs, c->gl);
  else
    pdl_launch(k_softmax_quant<kDecode>, g8, 256, 0, c->st, c->logits, c->probs, c->Bl, src,
               c->si(), c->intervals, c->cdf16, Bf, gs, nullptr);
  CK(cudaGetLastError());
  return EDPC_OK;
}

// -------------------------------------------------------------- backward

// g_up: gradient w.r.t. the block output [Bl][F]; writes the gradient w.r.t.
// the block input into g_in
static int mbrb_backward(edpc_ctx* c, const MbrbOffs& o, const MbrbBufs& b, const float* g_up,
                         float* g_in, float* GH, __half* guph) {
  const Layout& L = c->lay;
  const int Bl = c->Bl, F = L.F, H = o.H, K = L.K;
  const int64_t plane = (int64_t)Bl * H;
  if (c->h16) {
    const __half* x0h = reinterpret_cast<const __half*>(b.x0);
    const __half* ffh = reinterpret_cast<const __half*>(b.ff);
    const __half* Dh = reinterpret_cast<const __half*>(b.H);
    __half* GHh = reinterpret_cast<__half*>(GH);
    // guph: the fp16 copy of g_up, written by the dgrad that produced g_up (EpiStore2)
    if (mbrb_fused_enabled() && mbrb_fused_ok(F, H, K)) {
      // out-projection weight gradient on the side stream (needs g_up, ff);
      // out-proj dgrad + product rule + branch dgrad (+ its split reduction)
      // in one kernel (bit-identical to the three-launch path below); then the
      // branch weight gradients from the g_H it stored
      if (!c->wfuse) {  // needs only g_up and ff: overlaps the fused kernel
        CK(fork_aux(c));
        CK(wgrad_h(c, ffh, H, guph, F, 1, 0, o.out_w, 0, o.out_b));
      }
      {
        Scope sc(c, kRegGemm, c->st);
        const int st = mbrb_bwd_fused(guph, c->Wh + o.out_w, c->Wh + o.w0, o.wstride, Dh, GHh, Bl,
                                      H, c->gx0, c->st);
        if (st != EDPC_OK) return st;
      }
      CK(fork_aux(c));
      if (c->wfuse) CK(wgrad_h(c, ffh, H, guph, F, 1, 0, o.out_w, 0, o.out_b));
      CK(wgrad_h(c, x0h, F, GHh, H, K, plane, o.w0, o.wstride, o.b0));
    } else {
    // g_ff = g_up . out_w^T (out_w [H][F] = K-major B), epilogue -> g_H[z]
    {
      Scope sc(c, kRegGemm, c->st);
      TcShape s{Bl, H, F, 1, 1, kBatchNone, kBatchNone, 0, 1, 0, 0, 0};
      TcOperand a{guph, F, 0, 1}, bw{c->Wh + o.out_w, F, 0, 1};
      const int st = tc_gemm<false, false, true>(s, a, bw, EpiBwdActH{Dh, GHh, K, plane, H}, c->st);
      if (st != EDPC_OK) return st;
    }
    // weight gradients (and bias sums from fp32 g_up / fp16 g_H) on the side
    // stream -- after the branch dgrad's reads of W_z when they update W in
    // place (fused weight-gradient/Adam mode)
    if (!c->wfuse) {
      CK(fork_aux(c));
      CK(wgrad_h(c, ffh, H, guph, F, 1, 0, o.out_w, 0, o.out_b));
      CK(wgrad_h(c, x0h, F, GHh, H, K, plane, o.w0, o.wstride, o.b0));
    }
    // g_x0 = sum_z g_H[z] . W_z^T (W_z [F][H] = K-major B)
    CK(dgrad_h(c, GHh, H, K, plane, c->Wh + o.w0, o.wstride, F, c->gx0));
    if (c->wfuse) {
      CK(fork_aux(c));
      CK(wgrad_h(c, ffh, H, guph, F, 1, 0, o.out_w, 0, o.out_b));
      CK(wgrad_h(c, x0h, F, GHh, H, K, plane, o.w0, o.wstride, o.b0));
    }
    }
  } else {
  // g_ff = g_up . out_w^T, epilogue -> GH[z] (product rule + GeLU')
  CK(dgrad(c, g_up, F, 1, 0, wt(c) + o.out_w, 0, H, EpiBwdAct{b.H, GH, K, plane, H}));
  // weight gradients on the side stream (after the branch dgrad in the fused
  // weight-gradient/Adam mode, which updates W in place)
  if (!c->wfuse) {
    CK(fork_aux(c));
    CK(wgrad(c, b.ff, H, g_up, F, 1, 0, o.out_w, 0, o.out_b));
    CK(wgrad(c, b.x0, F, GH, H, K, plane, o.w0, o.wstride, o.b0));
  }
  // g_x0 = sum_z GH[z] . W_z^T
  CK(dgrad(c, GH, H, K, plane, wt(c) + o.w0, o.wstride, F, EpiStore{c->gx0, F}));
  if (c->wfuse) {
    CK(fork_aux(c));
    CK(wgrad(c, b.ff, H, g_up, F, 1, 0, o.out_w, 0, o.out_b));
    CK(wgrad(c, b.x0, F, GH, H, K, plane, o.w0, o.wstride, o.b0));
  }
  }
  // LN backward + residual, with the LN gain / bias gradient partials
  if (F <= kLnMaxF && c->g_count > 0) {
    int maxg = 0;
    for (int g = c->g_first; g < c->g_first + c->g_count; ++g)
      maxg = std::max(maxg, group_begin(g + 1, L.B) - group_begin(g, L.B));
    dim3 grid((unsigned)std::max(1, cdiv(maxg, kLnChunk)), (unsigned)c->g_count);
    Scope sc(c, kRegElem, c->st);
    pdl_launch(k_ln_bwd_fused, grid, 256, 0, c->st, c->gx0, b.xhat, b.rstd, c->W + o.ln_g, g_up, g_in, F,
                                            L.B, c->lane0, c->g_first, c->Gp, L.n_shared, o.ln_g,
                                            o.ln_b, c->ln_scratch, c->ln_tickets);
    CK(cudaGetLastError());
  } else {
    CK(colsum(c, c->gx0, F, 1, 0, b.xhat, o.ln_g, 0));
    CK(colsum(c, c->gx0, F, 1, 0, nullptr, o.ln_b, 0));
    Scope sc(c, kRegElem, c->st);
    pdl_launch(k_ln_bwd, (unsigned)cdiv(Bl, 8), 256, 0, c->st, c->gx0, b.xhat, b.rstd, c->W + o.ln_g, g_up,
                                                       g_in, F, Bl);
    CK(cudaGetLastError());
  }
  return EDPC_OK;
}

static int adam_range(edpc_ctx* c, int64_t off, int64_t len, cudaStream_t st, int nl = kNumGroups,
                      int64_t pstride = -1);
static bool early_adam(const edpc_ctx* c);
static int adam_span(edpc_ctx* c, int64_t lo, int64_t hi, cudaStream_t st);

static int backward(edpc_ctx* c, ByteCols src, float* nll, bool have_dlogits = false) {
  const Layout& L = c->lay;
  const int Bl = c->Bl, F = L.F, FP = L.FP;
  if (!have_dlogits) {
    Scope sc_(c, kRegElem, c->st);
    pdl_launch(k_dlogits, (unsigned)cdiv((int64_t)Bl * 256, 256), 256, 0, c->st, 
        c->probs, src, c->si(), Bl, (float)L.B, ldexpf(1.0f, c->gs_log2), c->gl, nll);
  }
  CK(cudaGetLastError());
  // head.  The weight gradients go to the side stream as early as possible
  // (before the dgrad that reads the same weights) -- except with the fused
  // weight-gradient/Adam kernels, which update W in place: then after it.
  if (!c->wfuse) {
    CK(fork_aux(c));
    CK(wgrad(c, c->x_global, F, c->gl, 256, 1, 0, L.head_w, 0, L.head_b));
  }
  if (c->h16)
    CK(dgrad(c, c->gl, 256, 1, 0, wt(c) + L.head_w, 0, F, EpiStore2{c->g_head, c->guph_g, F}));
  else
    CK(dgrad(c, c->gl, 256, 1, 0, wt(c) + L.head_w, 0, F, EpiStore{c->g_head, F}));
  if (c->wfuse) {
    CK(fork_aux(c));
    CK(wgrad(c, c->x_global, F, c->gl, 256, 1, 0, L.head_w, 0, L.head_b));
  }
  // global MBRB: d(x_global) -> d(x_lte)
  MbrbBufs gb{c->x_lte, c->g_xhat, c->g_rstd, c->g_x0, c->g_H, c->g_ff, c->x_global};
  EDPC_TRY(mbrb_backward(c, L.glo, gb, c->g_head, c->g_lte, c->GH_g, c->guph_g));
  if (c->wfuse) {  // global LN gain/bias (partials from k_ln_bwd_fused): complete
    CK(fork_aux(c));
    EDPC_TRY(adam_range(c, L.glo.ln_g, 2 * (int64_t)F, wst(c)));
  } else if (early_adam(c)) {  // global MBRB (its LN backward included) + head: complete
    CK(fork_aux(c));
    EDPC_TRY(adam_span(c, L.glo.ln_g, L.n_shared, c->st_aux));
  }
  // LTE up
  {
    if (!c->wfuse) {
      CK(fork_aux(c));
      CK(wgrad(c, c->mixed, FP, c->g_lte, F, 1, 0, L.up_w, 0, L.up_b));
    }
    CK(dgrad(c, c->g_lte, F, 1, 0, wt(c) + L.up_w, 0, FP, EpiStore{c->gmix, FP}));
    if (c->wfuse) {
      CK(fork_aux(c));
      CK(wgrad(c, c->mixed, FP, c->g_lte, F, 1, 0, L.up_w, 0, L.up_b));
    }
    // per-lane FDM: g_down with the old U, then U's Adam step (fused: U read once)
    {
      if (FP == 64 || FP == 128 || FP == 256) {
        const int lpw = 32 / std::min(32, FP / 4);
        const unsigned blocks = (unsigned)cdiv(cdiv(Bl, lpw), kFdmWarps);
        auto run = [&](auto kern, cudaStream_t st) {
          Scope sc_(c, kRegFdmBwd, st);
          pdl_launch(kern, blocks, 32 * kFdmWarps, 0, st, c->down, c->gmix, c->U, c->Um, c->Uv,
                     c->gdown, Bl, c->si(), c->adam, c->cfg.beta1, c->cfg.beta2,
                     ldexpf(1.0f, -c->gs_log2));
        };
        // (a split variant -- FDM backward on the main stream, U's Adam pass on
        // the side stream -- measured 3% slower at C2 in round 1 and 6% slower
        // in round 2 (9.44 -> 8.89 MB/s A/B): the passes compete for HBM and U
        // is read twice)
        if (FP == 64)
          run(k_fdm_bwd_adam_v<64>, c->st);
        else if (FP == 128)
          run(k_fdm_bwd_adam_v<128>, c->st);
        else
          run(k_fdm_bwd_adam_v<256>, c->st);
      } else {
        Scope sc_(c, kRegFdmBwd, c->st);
        pdl_launch(k_fdm_bwd_adam, (unsigned)cdiv(Bl, 8), 256, 0, c->st, 
            c->down, c->gmix, c->U, c->Um, c->Uv, c->gdown, FP, Bl, c->si(), c->adam,
            c->cfg.beta1, c->cfg.beta2, ldexpf(1.0f, -c->gs_log2));
      }
    }
    CK(cudaGetLastError());
    // LTE down
    if (!c->wfuse) {
      CK(fork_aux(c));
      CK(wgrad(c, c->x_local, F, c->gdown, FP, 1, 0, L.down_w, 0, L.down_b));
    }
    if (c->h16)
      CK(dgrad(c, c->gdown, FP, 1, 0, wt(c) + L.down_w, 0, F, EpiStore2{c->g_loc, c->guph_l, F}));
    else
      CK(dgrad(c, c->gdown, FP, 1, 0, wt(c) + L.down_w, 0, F, EpiStore{c->g_loc, F}));
    if (c->wfuse) {
      CK(fork_aux(c));
      CK(wgrad(c, c->x_local, F, c->gdown, FP, 1, 0, L.down_w, 0, L.down_b));
    }
  }
  if (!c->wfuse && early_adam(c)) {  // LTE down + up
    CK(fork_aux(c));
    EDPC_TRY(adam_span(c, L.down_w, L.glo.ln_g, c->st_aux));
  }
  // local MBRB: d(x_local) -> d(x_emb) (gradient w.r.t. the embedded context)
  MbrbBufs lb{c->x_emb, c->l_xhat, c->l_rstd, c->l_x0, c->l_H, c->l_ff, c->x_local};
  EDPC_TRY(mbrb_backward(c, L.loc, lb, c->g_loc, c->g_emb, c->GH_l, c->guph_l));
  if (!c->wfuse && early_adam(c)) {  // local MBRB: complete; overlaps the embedding scatter-add
    CK(fork_aux(c));
    EDPC_TRY(adam_span(c, L.loc.ln_g, L.down_w, c->st_aux));
  }
  // embedding scatter-add as per-group partials
  if (c->n_chunks > 0) {
    {
      Scope sc_(c, kRegEmbed, c->st);
      pdl_launch(k_embed_grad_chunks, (unsigned)c->n_chunks, 256, 0, c->st, src, c->si(), L.T, L.DE, F,
                                                                    c->g_emb, c->chunk_tab, c->emb_sub);
    }
    CK(cudaGetLastError());
    dim3 gr((unsigned)cdiv(256 * L.DE, 256), (unsigned)c->g_count);
    {
      Scope sc_(c, kRegEmbed, c->st);
      pdl_launch(k_embed_grad_reduce, gr, 256, 0, c->st, c->emb_sub, c->grp_chunks, L.DE, c->Gp,
                                                 L.n_shared, L.emb);
    }
    CK(cudaGetLastError());
  }
  CK(join_aux(c));
  return EDPC_OK;
}

// ------------------------------------------------ shared-parameter Adam
//
// One context holding all 8 lane groups: grad = the 8-leaf canonical tree
// over its partials, Adam over every shared parameter.
//
// G > 1 contexts (one per GPU, or several on one GPU through dist.ShardSet),
// rank r owning the 8/G groups [r*8/G, (r+1)*8/G) -- the sharded optimizer of
// SURVEY.md §8e:
//   1. k_group_tree: the rank's subtree sum of its groups, into its first
//      group's partial slot (skipped when 8/G == 1);
//   2. slice exchange: the shared parameters are cut into G slices; rank j's
//      subtree sum of slice r goes to rank r (NCCL send/recv, or peer copies
//      via edpc_partials_pull), landing in slot j*8/G of r's partial buffer;
//   3. k_adam_shared<G> on the owned slice: the G-leaf tree over the subtree
//      sums (= the 8-leaf tree, bit for bit) then Adam; m, v are only ever
//      touched on the owned slice;
//   4. all-gather of the updated fp32 weights and their fp16 shadow (NCCL
//      in place, or edpc_weights_pull).
// Per step each GPU sends (G-1)/G of one partial and receives (G-1)/G of the
// weights, instead of all-gathering 8/G full partials per rank.

static int shard_count(const edpc_ctx* c) {
  return c->g_count > 0 && c->g_count < kNumGroups ? kNumGroups / c->g_count : 1;
}
static int shard_rank(const edpc_ctx* c) {
  return shard_count(c) > 1 ? c->g_first / c->g_count : 0;
}
static int64_t shard_slice(const edpc_ctx* c) {
  const int G = shard_count(c);
  return (cdiv(c->lay.n_shared, (int64_t)G) + 63) / 64 * 64;
}
// owned parameter range [*off, *off + *len) of shard r
static void shard_range(const edpc_ctx* c, int r, int64_t* off, int64_t* len) {
  const int64_t s = shard_slice(c), P = c->lay.n_shared;
  *off = std::min<int64_t>(P, (int64_t)r * s);
  *len = std::min<int64_t>(P, (int64_t)(r + 1) * s) - *off;
}

template <int NL>
static void adam_launch(edpc_ctx* c, int blocks, cudaStream_t st, int64_t off, int64_t len,
                        int64_t pstride) {
  pdl_launch(k_adam_shared<NL>, blocks, 256, 0, st, c->W + off, c->M + off, c->V + off,
             c->Gp + off, len, pstride, c->si(), c->adam, c->cfg.beta1, c->cfg.beta2,
             ldexpf(1.0f, -c->gs_log2), c->h16 ? c->Wh + off : nullptr,
             c->rt ? c->Wt + off : nullptr);
}

// Adam over shared params [off, off + len) on stream st; nl leaves at stride
// pstride (8 lane groups, or G subtree sums)
static int adam_range(edpc_ctx* c, int64_t off, int64_t len, cudaStream_t st, int nl,
                      int64_t pstride) {
  if (len <= 0) return EDPC_OK;
  if (pstride < 0) pstride = c->lay.n_shared;
  const int blocks = (int)std::min<int64_t>(cdiv(len, 256), 148 * 8);
  {
    Scope sc_(c, kRegAdam, st);
    switch (nl) {
      case 1: adam_launch<1>(c, blocks, st, off, len, pstride); break;
      case 2: adam_launch<2>(c, blocks, st, off, len, pstride); break;
      case 4: adam_launch<4>(c, blocks, st, off, len, pstride); break;
      case 8: adam_launch<8>(c, blocks, st, off, len, pstride); break;
      default: set_error("bad leaf count"); return EDPC_ERR_INVALID;
    }
  }
  CK(cudaGetLastError());
  return EDPC_OK;
}

// Early Adam: with all 8 lane groups in this context (no exchange before the
// optimizer), the global-MBRB weights + head, the LTE projections and the
// local MBRB are updated on the side stream as soon as their gradients are
// complete and the main stream has finished reading them; only the embedding
// (256 x d_e parameters) is left for the end of the step.
static bool early_adam(const edpc_ctx* c) {
  return c->g_count == kNumGroups && !c->comm && aux_enabled();
}

// step 1 (sharded): subtree sum of the local groups into slot g_first
static int group_tree(edpc_ctx* c) {
  if (shard_count(c) < 2 || c->g_count < 2) return EDPC_OK;
  const int64_t P = c->lay.n_shared;
  const int blocks = (int)std::min<int64_t>(cdiv(P, 256), 148 * 8);
  float* base = c->Gp + (size_t)c->g_first * P;
  {
    Scope sc_(c, kRegAdam, c->st);
    if (c->g_count == 2)
      pdl_launch(k_group_tree<2>, blocks, 256, 0, c->st, base, P, P);
    else if (c->g_count == 4)
      pdl_launch(k_group_tree<4>, blocks, 256, 0, c->st, base, P, P);
    else {
      set_error("bad lane-group share");
      return EDPC_ERR_INVALID;
    }
  }
  CK(cudaGetLastError());
  return EDPC_OK;
}

// Adam over [lo, hi) of the shared parameters with the right leaf count per
// sub-range: the LN gains/biases and the embedding always have 8 lane-group
// partials; the weight-gradient ranges have 2 subtree partials (slots 0, 4)
// in subtree mode, else 8.
static int adam_span(edpc_ctx* c, int64_t lo, int64_t hi, cudaStream_t st) {
  const Layout& L = c->lay;
  const int w = c->wsub ? 2 : kNumGroups;
  const struct {
    int64_t a, b;
    int nl;
  } seg[] = {{0, L.loc.w0, kNumGroups},       // embedding + local LN
             {L.loc.w0, L.glo.ln_g, w},       // local MBRB weights, LTE
             {L.glo.ln_g, L.glo.w0, kNumGroups},  // global LN
             {L.glo.w0, L.n_shared, w}};      // global MBRB weights, head
  for (const auto& s : seg) {
    const int64_t a = std::max(lo, s.a), b = std::min(hi, s.b);
    if (a < b)
      EDPC_TRY(adam_range(c, a, b - a, st, s.nl,
                          s.nl == 2 ? (int64_t)4 * L.n_shared : (int64_t)L.n_shared));
  }
  return EDPC_OK;
}

static int adam_shared(edpc_ctx* c) {
  const Layout& L = c->lay;
  const int G = shard_count(c);
  if (G > 1) {  // step 3 (sharded): owned slice, G-leaf tree over subtree sums
    int64_t off, len;
    shard_range(c, shard_rank(c), &off, &len);
    return adam_range(c, off, len, c->st, G, (int64_t)c->g_count * L.n_shared);
  }
  // fused weight gradients: only the embedding and the local LN (contiguous)
  // are left; the global LN went on the side stream after its backward
  if (c->wfuse) return adam_range(c, 0, L.loc.ln_g + 2 * (int64_t)L.F, c->st);
  if (early_adam(c)) return adam_span(c, 0, L.loc.ln_g, c->st);  // the embedding
  return adam_span(c, 0, L.n_shared, c->st);
}

static int nccl_fail(const char* what, ncclResult_t r) {
  set_error(std::string(what) + ": " + nccl().getErrorString(r));
  return EDPC_ERR_CUDA;
}

// step 2 over NCCL: rank j's subtree sum of slice r -> rank r, slot j*8/G
static int exchange_slices(edpc_ctx* c) {
  if (!c->comm || c->nranks < 2) return EDPC_OK;
  const int G = c->nranks, r = c->rank;
  const size_t P = (size_t)c->lay.n_shared, gc = (size_t)c->g_count;
  int64_t ro, rl;
  shard_range(c, r, &ro, &rl);
  ncclResult_t e = nccl().groupStart();
  if (e != ncclSuccess) return nccl_fail("ncclGroupStart", e);
  for (int j = 0; j < G && e == ncclSuccess; ++j) {
    if (j == r) continue;
    int64_t jo, jl;
    shard_range(c, j, &jo, &jl);
    if (jl > 0) e = nccl().send(c->Gp + r * gc * P + jo, (size_t)jl, ncclFloat, j, c->comm, c->st);
    if (e == ncclSuccess && rl > 0)
      e = nccl().recv(c->Gp + j * gc * P + ro, (size_t)rl, ncclFloat, j, c->comm, c->st);
  }
  ncclResult_t e2 = nccl().groupEnd();
  if (e != ncclSuccess) return nccl_fail("ncclSend/ncclRecv", e);
  if (e2 != ncclSuccess) return nccl_fail("ncclGroupEnd", e2);
  return EDPC_OK;
}

// step 4 over NCCL: in-place all-gather of the owned weight slices (fp32 and
// the fp16 shadow); W / Wh are padded to G equal slices
static int exchange_weights(edpc_ctx* c) {
  if (!c->comm || c->nranks < 2) return EDPC_OK;
  const size_t s = (size_t)shard_slice(c), r = (size_t)c->rank;
  ncclResult_t e = nccl().allGather(c->W + r * s, c->W, s, ncclFloat, c->comm, c->st);
  if (e != ncclSuccess) return nccl_fail("ncclAllGather(W)", e);
  if (c->h16) {
    e = nccl().allGather(c->Wh + r * s, c->Wh, s, ncclHalf, c->comm, c->st);
    if (e != ncclSuccess) return nccl_fail("ncclAllGather(Wh)", e);
  }
  if (c->rt) {
    e = nccl().allGather(c->Wt + r * s, c->Wt, s, ncclFloat, c->comm, c->st);
    if (e != ncclSuccess) return nccl_fail("ncclAllGather(Wt)", e);
  }
  return EDPC_OK;
}

// steps 1-4 after backward()
static int optimizer_step(edpc_ctx* c) {
  EDPC_TRY(group_tree(c));
  EDPC_TRY(exchange_slices(c));
  EDPC_TRY(adam_shared(c));
  EDPC_TRY(exchange_weights(c));
  return EDPC_OK;
}

// One model step at lane column d_i + step_off (Adam count d_t + step_off);
// advance > 0: the step ends by moving d_i / d_t on by `advance` (a captured
// graph of kGraphSteps steps advances once, by kGraphSteps, at its end).
static int model_step(edpc_ctx* c, int mode, int advance = 1) {
  ByteCols src = c->lanes_src();
  EDPC_TRY(forward(c, src));
  EDPC_TRY(softmax_quant(c, mode, src));
  if (mode == kDecode) {
    Scope sc(c, kRegDecode, c->st);
    pdl_launch(k_decode_column, (unsigned)cdiv(c->Sl, 4), 128, 0, c->st, 
        c->mat, c->L, c->si(), c->spl, c->Sl, c->cdf16, false, c->dec_state, c->payload,
        c->pay_off, c->bit_len, c->dec_err);
    CK(cudaGetLastError());
  }
  EDPC_TRY(backward(c, src, nullptr, mode == kEncode));
  EDPC_TRY(optimizer_step(c));
  if (advance > 0) {
    Scope sc_(c, kRegElem, c->st);
    pdl_launch(k_step_advance, 1, 1, 0, c->st, c->d_i, c->d_t, advance);
  }
  CK(cudaGetLastError());
  return EDPC_OK;
}

// CUDA graphs: kGraphSteps consecutive model steps are captured once per
// mode and replayed; the step index lives in device memory (d_i / d_t) and is
// advanced by the last kernel of each step, so replays need no host input.
constexpr int kGraphSteps = 16;

static bool graphs_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("EDPC_GRAPHS");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

static int run_model_steps(edpc_ctx* c, int64_t n, int mode) {
  const bool use_graph = graphs_enabled() && !c->prof.on && !sync_debug();
  if (use_graph && n >= kGraphSteps) {
    cudaGraphExec_t& ge = c->graph[mode == kDecode ? 1 : 0];
    if (!ge) {
      cudaGraph_t g = nullptr;
      CK(cudaStreamBeginCapture(c->st, cudaStreamCaptureModeThreadLocal));
      int st = EDPC_OK;
      for (int k = 0; k < kGraphSteps && st == EDPC_OK; ++k) {
        c->step_off = k;
        st = model_step(c, mode, k == kGraphSteps - 1 ? kGraphSteps : 0);
      }
      c->step_off = 0;
      cudaError_t e = cudaStreamEndCapture(c->st, &g);
      if (st != EDPC_OK) {
        if (g) cudaGraphDestroy(g);
        return st;
      }
      CK(e);
      if (c->l2win.num_bytes) {  // the U window on every kernel node of the step graph
        size_t nn = 0;
        CK(cudaGraphGetNodes(g, nullptr, &nn));
        std::vector<cudaGraphNode_t> nodes(nn);
        CK(cudaGraphGetNodes(g, nodes.data(), &nn));
        cudaKernelNodeAttrValue v{};
        v.accessPolicyWindow = c->l2win;
        for (auto nd : nodes) {
          cudaGraphNodeType ty;
          CK(cudaGraphNodeGetType(nd, &ty));
          if (ty == cudaGraphNodeTypeKernel)
            CK(cudaGraphKernelNodeSetAttribute(nd, cudaKernelNodeAttributeAccessPolicyWindow, &v));
        }
      }
      e = cudaGraphInstantiate(&ge, g, 0);
      cudaGraphDestroy(g);
      CK(e);
    }
    while (n >= kGraphSteps) {
      CK(cudaGraphLaunch(ge, c->st));
      n -= kGraphSteps;
    }
  }
  for (; n > 0; --n) EDPC_TRY(model_step(c, mode));
  return EDPC_OK;
}

// U (the per-lane FDM matrices, read by the LTE forward and read + rewritten
// by the FDM backward/Adam every step: 67 MB at C2) is the one large array
// re-read within a step and across steps.  When it fits one access policy
// window (<= the 79 MB persisting maximum on B200) a window over it marks a
// fraction of its lines persisting (a set-aside of that size).  Measured on
// C2 (compress MB/s): fraction 0 8.80, 0.15 8.89, 0.3 8.91, 0.5 8.75, 1.0 7.81
// -- the GEMMs need the rest of L2.  Numerics-neutral; EDPC_L2_PERSIST=<fraction>
// overrides the default 0.3 (0 turns it off).
static void l2_persist_setup(edpc_ctx* c, size_t bytes) {
  const char* e = getenv("EDPC_L2_PERSIST");
  const double frac = e ? atof(e) : 0.3;
  if (!(frac > 0.0)) return;
  int max_persist = 0, max_win = 0;
  if (cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, c->device) !=
          cudaSuccess ||
      cudaDeviceGetAttribute(&max_win, cudaDevAttrMaxAccessPolicyWindowSize, c->device) !=
          cudaSuccess) {
    cudaGetLastError();
    return;
  }
  if (bytes == 0 || bytes > (size_t)max_persist || bytes > (size_t)max_win) return;
  size_t cur = 0;
  cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
  const size_t aside = (size_t)(std::min(frac, 1.0) * (double)bytes);
  if (cur < aside && cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, aside) != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  c->l2win.base_ptr = c->U;
  c->l2win.num_bytes = bytes;
  c->l2win.hitRatio = (float)std::min(frac, 1.0);
  c->l2win.hitProp = cudaAccessPropertyPersisting;
  c->l2win.missProp = cudaAccessPropertyStreaming;
  cudaStreamAttrValue v{};
  v.accessPolicyWindow = c->l2win;
  if (cudaStreamSetAttribute(c->st, cudaStreamAttributeAccessPolicyWindow, &v) != cudaSuccess) {
    cudaGetLastError();
    c->l2win.num_bytes = 0;
  }
}

static int set_step(edpc_ctx* c, int64_t i, int64_t t) {
  int64_t h[2] = {i, t};
  CK(cudaMemcpyAsync(c->d_i, &h[0], 8, cudaMemcpyHostToDevice, c->st));
  CK(cudaMemcpyAsync(c->d_t, &h[1], 8, cudaMemcpyHostToDevice, c->st));
  return EDPC_OK;
}

// Context buffers come from the device's default stream-ordered pool, with the
// release threshold lifted so freed contexts keep their memory for the next
// one (back-to-back compress/decompress calls skip cudaMalloc/cudaFree, whose
// first-touch mapping and implicit device syncs cost 0.1-1.3 s per context at
// C2/C3 sizes); `edpc_trim_pool` hands it back.  Peers that can reach the
// device get pool access (the sharded optimizer's peer pulls).
static void pool_setup(int device) {
  static std::mutex mu;
  static std::vector<bool> done;
  std::lock_guard<std::mutex> g(mu);
  if (device < 0) return;
  if ((int)done.size() <= device) done.resize(device + 1, false);
  if (done[device]) return;
  done[device] = true;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) != cudaSuccess) return;
  uint64_t keep = UINT64_MAX;
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  int n = 0;
  cudaGetDeviceCount(&n);
  for (int p = 0; p < n; ++p) {
    int ok = 0;
    if (p == device || cudaDeviceCanAccessPeer(&ok, p, device) != cudaSuccess || !ok) continue;
    cudaMemAccessDesc d{};
    d.location.type = cudaMemLocationTypeDevice;
    d.location.id = p;
    d.flags = cudaMemAccessFlagsProtReadWrite;
    cudaMemPoolSetAccess(pool, &d, 1);
  }
  cudaGetLastError();
}

static int launch_encoder(edpc_ctx* c, int64_t upto) {
  if (upto <= c->enc_upto) return EDPC_OK;
  CK(cudaEventRecord(c->ev, c->st));
  CK(cudaStreamWaitEvent(c->st_enc, c->ev, 0));
  Scope sc(c, kRegEncode, c->st_enc);
  pdl_launch(k_encode_columns, (unsigned)cdiv(c->Sl, 64), 64, 0, c->st_enc, 
      c->intervals, c->Bl, c->spl, c->Sl, c->enc_upto, upto, c->enc_state, c->enc_words,
      c->enc_cap_words);
  CK(cudaGetLastError());
  c->enc_upto = upto;
  return EDPC_OK;
}

}  // namespace edpc

// ================================================================== C ABI

extern "C" {

int edpc_has_tcgen05(void) { return tc_compiled() ? 1 : 0; }

int edpc_ctx_create(const edpc_config* cfg, int32_t segments, int64_t original_len,
                    int32_t device, int32_t lane_begin, int32_t lane_count, edpc_ctx** out) {
  return edpc_ctx_create_ex(cfg, segments, original_len, device, lane_begin, lane_count, -1, out);
}

int edpc_ctx_create_ex(const edpc_config* cfg, int32_t segments, int64_t original_len,
                       int32_t device, int32_t lane_begin, int32_t lane_count, int32_t numerics,
                       edpc_ctx** out) {
  EDPC_CHECK_ARG(out, "null out");
  EDPC_CHECK_ARG(numerics >= -1 && numerics <= kNumericsMask, "unknown numerics flags");
  *out = nullptr;
  EDPC_TRY(check_cfg(cfg));
  EDPC_CHECK_ARG(segments >= 1 && cfg->lanes % segments == 0,
                 "segments must divide lanes");
  EDPC_CHECK_ARG(original_len >= 0, "negative length");
  EDPC_CHECK_ARG(lane_begin >= 0 && lane_count >= 1 && lane_begin + lane_count <= cfg->lanes,
                 "bad lane range");
  const int spl = cfg->lanes / segments;
  EDPC_CHECK_ARG(lane_begin % spl == 0 && lane_count % spl == 0,
                 "lane range must cover whole segments");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    set_error("no CUDA device available (the B200 path has no CPU fallback)");
    return EDPC_ERR_CUDA;
  }
  EDPC_CHECK_ARG(device >= 0 && device < ndev, "device ordinal out of range");
  EDPC_CUDA_TRY(cudaSetDevice(device));

  edpc_ctx* c = new edpc_ctx();
  c->cfg = *cfg;
  c->lay.build(*cfg);
  c->device = device;
  c->Bl = lane_count;
  c->lane0 = lane_begin;
  c->S = segments;
  c->spl = spl;
  c->Sl = lane_count / spl;
  c->seg0 = lane_begin / spl;
  c->n = original_len;
  c->L = original_len ? (original_len + cfg->lanes - 1) / cfg->lanes : 0;
  // local lane groups: group g belongs to the device holding its first lane
  // (multi-device callers split B on group boundaries, see dist.py)
  c->g_first = -1;
  c->g_count = 0;
  for (int g = 0; g < kNumGroups; ++g) {
    int b0 = group_begin(g, cfg->lanes);
    if (b0 >= lane_begin && b0 < lane_begin + lane_count) {
      if (c->g_first < 0) c->g_first = g;
      c->g_count++;
    }
  }
  if (c->g_first < 0) c->g_first = 0;
  {
    double b1 = cfg->beta1, b2 = cfg->beta2;
    c->adam.lr = (float)cfg->lr;
    c->adam.b1 = (float)b1;
    c->adam.b2 = (float)b2;
    c->adam.k1 = (float)(1.0 - b1);
    c->adam.k2 = (float)(1.0 - b2);
    c->adam.eps = (float)cfg->adam_eps;
  }
  // Numerics policy (recorded in the container; by default a function of the
  // config only).  TF32 tensor-core GEMMs when the container has >=
  // kTf32MinLanes lanes: the per-step gradient averages over enough lanes
  // that TF32 operand rounding does not move the compression ratio (C2-mini,
  // B=4096: +0.07% vs the fp64 reference); below that (e.g. config 1, B=64)
  // TF32 moved the ratio by -1.35%..+0.84% over three streams, fp32 by at
  // most 0.34%, so small-lane containers use the fp32 GEMMs.  fp16 operands
  // for the MBRB GEMMs on the tensor-core path whenever the shapes tile (k = 2,
  // F and the lane groups multiples of 64 for the fp16 k-blocks, H multiple
  // of 128).  The fused LTE forward at paper dims.  numerics >= 0 (the
  // decoder replaying a container's recorded flags, or a test) forces the
  // flags; infeasible combinations are refused.
  {
    const Layout& L = c->lay;
    const int glanes = L.B / kNumGroups;
    const bool tc_ok_cfg = tc_compiled();
    const bool h16_ok = L.K == 2 && L.F % 64 == 0 && L.HL % 128 == 0 && L.HG % 128 == 0 &&
                        L.B % kNumGroups == 0 && glanes % 64 == 0;
    if (numerics < 0) {
      c->use_tc = tc_ok_cfg && cfg->lanes >= kTf32MinLanes;
      c->h16 = c->use_tc && h16_ok;
      c->lte_fwd = lte_fused_possible(c);
      c->rt = c->use_tc;
    } else {
      c->use_tc = (numerics & kNumTc) != 0;
      c->h16 = (numerics & kNumF16) != 0;
      c->lte_fwd = (numerics & kNumLteFused) != 0;
      c->rt = (numerics & kNumRndTf32) != 0;
      const bool ok = (!c->use_tc || tc_ok_cfg) && (!c->h16 || (c->use_tc && h16_ok)) &&
                      (!c->lte_fwd || lte_fused_possible(c)) && (!c->rt || c->use_tc);
      if (!ok) {
        delete c;
        set_error("numerics flags " + std::to_string(numerics) +
                  " cannot run for this config / build");
        return EDPC_ERR_INVALID;
      }
    }
    int k = 0;
    while ((2 << k) <= L.B) ++k;  // 2^k <= B < 2^(k+1)
    c->gs_log2 = k;
  }

  // fused weight-gradient + Adam kernels (wgrad_adam.cuh): the tensor-core
  // path with all 8 lane groups in this context, 64-lane-multiple groups,
  // every weight gradient N a multiple of the 64-column tile and 16-byte
  // aligned weights.  Numerics-neutral (bit-identical to the partials +
  // k_adam_shared path) but OFF by default: one CTA walking all 8 groups of
  // a tile is latency-bound in its operand pipeline (ncu: ~60 us per tile,
  // C2 6.0 vs 8.8 MB/s) -- 8x fewer CTAs than the partial GEMMs, each 8x
  // longer.  EDPC_WGRAD_FUSED=1 selects it (experiments / A-B tests).
  {
    const Layout& L = c->lay;
    const char* e = getenv("EDPC_WGRAD_FUSED");
    bool ok = (e && e[0] == '1') && c->use_tc && c->g_count == kNumGroups && L.B % kNumGroups == 0 &&
              (L.B / kNumGroups) % 64 == 0;
    for (int n : {L.F, L.FP, L.HL, L.HG, 256}) ok = ok && n % 64 == 0;
    for (int64_t o : {L.loc.w0, L.loc.wstride, L.loc.out_w, L.glo.w0, L.glo.wstride, L.glo.out_w,
                      L.down_w, L.up_w, L.head_w})
      ok = ok && o % 8 == 0;
    c->wfuse = ok;
    // subtree weight gradients: the same geometry conditions.  Numerics-
    // neutral but OFF by default: its CTAs walk 4 groups through a 128-wide
    // tile, twice the k-blocks of the 256-wide per-group GEMMs, and the
    // per-CTA operand pipeline (~1 k-block per us) is what bounds both (ncu:
    // global branch 75.7 vs 42.6 us; C2 7.4 vs 8.8 MB/s).  EDPC_WGRAD_SUBTREE=1.
    const char* e2 = getenv("EDPC_WGRAD_SUBTREE");
    bool sok = (e2 && e2[0] == '1') && c->use_tc && c->g_count == kNumGroups &&
               L.B % kNumGroups == 0 && (L.B / kNumGroups) % 64 == 0;
    for (int n : {L.F, L.FP, L.HL, L.HG, 256}) sok = sok && n % 64 == 0;
    c->wsub = sok && !c->wfuse;
  }
  auto fail = [&](int code) {
    delete c;
    return code;
  };
  pool_setup(c->device);
  if (cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->st_enc, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev, cudaEventDisableTiming) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->st_aux, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->st_h2d, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_h2d, cudaEventDisableTiming) != cudaSuccess) {
    set_error("stream/event creation failed");
    return fail(EDPC_ERR_CUDA);
  }
  const Layout& L = c->lay;
  const int Bl = c->Bl;
  const int64_t F = L.F, FP = L.FP;
#define A_(p, n)                        \
  do {                                  \
    int _r = c->alloc(&(p), (n));       \
    if (_r != EDPC_OK) return fail(_r); \
  } while (0)
  // W, M, V in one allocation at a fixed element distance (one TMA map reaches
  // all three from the fused weight-gradient/Adam kernel); W padded for the
  // in-place all-gather of equal slices
  c->arr = (L.n_shared + kShardPad + 63) / 64 * 64;
  A_(c->W, 3 * c->arr);
  c->M = c->W + c->arr;
  c->V = c->M + c->arr;
  A_(c->Gp, (int64_t)kNumGroups * L.n_shared);
  A_(c->U, (int64_t)Bl * L.fdm);
  l2_persist_setup(c, (size_t)Bl * L.fdm * sizeof(float));
  A_(c->Um, (int64_t)Bl * L.fdm);
  A_(c->Uv, (int64_t)Bl * L.fdm);
  A_(c->mat, (int64_t)Bl * std::max<int64_t>(c->L, 1));
  A_(c->scratch, (int64_t)Bl * (L.T + 1));
  A_(c->d_i, 2);
  A_(c->d_t, 2);
  A_(c->x_emb, Bl * F);
  A_(c->l_xhat, Bl * F);
  A_(c->l_rstd, Bl);
  A_(c->l_x0, Bl * F);
  A_(c->l_H, (int64_t)L.K * Bl * L.HL);
  A_(c->l_ff, (int64_t)Bl * L.HL);
  A_(c->x_local, Bl * F);
  A_(c->down, Bl * FP);
  A_(c->mixed, Bl * FP);
  A_(c->x_lte, Bl * F);
  A_(c->g_xhat, Bl * F);
  A_(c->g_rstd, Bl);
  A_(c->g_x0, Bl * F);
  A_(c->g_H, (int64_t)L.K * Bl * L.HG);
  A_(c->g_ff, (int64_t)Bl * L.HG);
  A_(c->x_global, Bl * F);
  A_(c->logits, (int64_t)Bl * 256);
  A_(c->probs, (int64_t)Bl * 256);
  A_(c->nll, Bl);
  A_(c->gl, (int64_t)Bl * 256);
  A_(c->g_head, Bl * F);
  A_(c->g_lte, Bl * F);
  A_(c->g_loc, Bl * F);
  A_(c->g_emb, Bl * F);
  A_(c->GH_g, (int64_t)L.K * Bl * L.HG);
  A_(c->GH_l, (int64_t)L.K * Bl * L.HL);
  if (c->rt) A_(c->Wt, L.n_shared + kShardPad);
  if (c->h16) {
    A_(c->Wh, L.n_shared + kShardPad);
    A_(c->guph_l, Bl * F);
    A_(c->guph_g, Bl * F);
  }
  A_(c->gx0, Bl * F);
  A_(c->gmix, Bl * FP);
  A_(c->gdown, Bl * FP);
  A_(c->ws, (int64_t)kSplitK * Bl * 256);
  A_(c->ln_scratch, (int64_t)kNumGroups * (cdiv(Bl, kLnChunk) + 1) * 2 * F);
  A_(c->ln_tickets, kNumGroups);
  // embedding-gradient chunks: <= 64 lanes (and <= 4096 context bytes) each,
  // never straddling a lane group
  {
    const int chunk = std::max(1, std::min(kEmbChunkLanes, 4096 / L.T));
    std::vector<int> tab, grp;
    int k = 0;
    for (int g = c->g_first; g < c->g_first + c->g_count; ++g) {
      int b0 = group_begin(g, L.B) - c->lane0, b1 = group_begin(g + 1, L.B) - c->lane0;
      int k0 = k;
      for (int b = b0; b < b1; b += chunk) {
        tab.push_back(g);
        tab.push_back(b);
        tab.push_back(std::min(b + chunk, b1));
        ++k;
      }
      grp.push_back(g);
      grp.push_back(k0);
      grp.push_back(k);
    }
    c->n_chunks = k;
    A_(c->chunk_tab, (int64_t)std::max<size_t>(tab.size(), 3));
    A_(c->grp_chunks, (int64_t)std::max<size_t>(grp.size(), 3));
    A_(c->emb_sub, (int64_t)std::max(k, 1) * 256 * L.DE);
    if (!tab.empty() &&
        cudaMemcpy(c->chunk_tab, tab.data(), tab.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess)
      return fail(EDPC_ERR_CUDA);
    if (!grp.empty() &&
        cudaMemcpy(c->grp_chunks, grp.data(), grp.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess)
      return fail(EDPC_ERR_CUDA);
  }
  // coder buffers: 18 bits per symbol worst case (coder.py:269-270) + slack
  A_(c->intervals, std::max<int64_t>(c->L, 1) * Bl);
  A_(c->cdf16, (int64_t)Bl * 256);
  A_(c->enc_state, 4 * (int64_t)c->Sl);
  A_(c->dec_state, 4 * (int64_t)c->Sl);
  c->enc_cap_words = (18 * (int64_t)c->spl * std::max<int64_t>(c->L, 1) + 128) / 32 + 2;
  A_(c->enc_words, c->enc_cap_words * c->Sl);
  A_(c->pay_off, c->Sl + 1);
  A_(c->bit_len, c->Sl);
  A_(c->dec_err, c->Sl);
#undef A_
  // zero state: Adam moments, encoders (low=0, high=2^32-1), error flags
  cudaMemsetAsync(c->M, 0, L.n_shared * 4, c->st);
  cudaMemsetAsync(c->V, 0, L.n_shared * 4, c->st);
  cudaMemsetAsync(c->Um, 0, (int64_t)Bl * L.fdm * 4, c->st);
  cudaMemsetAsync(c->Uv, 0, (int64_t)Bl * L.fdm * 4, c->st);
  cudaMemsetAsync(c->Gp, 0, (int64_t)kNumGroups * L.n_shared * 4, c->st);
  cudaMemsetAsync(c->enc_words, 0, c->enc_cap_words * c->Sl * 4, c->st);
  cudaMemsetAsync(c->dec_err, 0, c->Sl * 4, c->st);
  cudaMemsetAsync(c->ln_tickets, 0, kNumGroups * 4, c->st);
  {
    std::vector<int64_t> es(4 * (size_t)c->Sl);
    for (int s = 0; s < c->Sl; ++s) {
      es[4 * s + 0] = 0;
      es[4 * s + 1] = (int64_t)kMask32;
      es[4 * s + 2] = 0;
      es[4 * s + 3] = 0;
    }
    cudaMemcpy(c->enc_state, es.data(), es.size() * 8, cudaMemcpyHostToDevice);
  }
  if (cudaStreamSynchronize(c->st) != cudaSuccess) {
    set_error("context init failed");
    return fail(EDPC_ERR_CUDA);
  }
  *out = c;
  return EDPC_OK;
}

int edpc_ctx_destroy(edpc_ctx* ctx) {
  if (ctx) {
    cudaSetDevice(ctx->device);
    delete ctx;
  }
  return EDPC_OK;
}

int edpc_ctx_numerics(edpc_ctx* c, int32_t* flags) {
  EDPC_CHECK_ARG(c && flags, "null argument");
  *flags = (c->use_tc ? kNumTc : 0) | (c->h16 ? kNumF16 : 0) | (c->lte_fwd ? kNumLteFused : 0) |
           (c->rt ? kNumRndTf32 : 0);
  return EDPC_OK;
}

int edpc_ctx_info(edpc_ctx* c, int64_t* lane_len, int64_t* n_params, int64_t* n_shared) {
  EDPC_CHECK_ARG(c, "null ctx");
  if (lane_len) *lane_len = c->L;
  if (n_params) *n_params = c->lay.n_ref;
  if (n_shared) *n_shared = c->lay.n_shared;
  return EDPC_OK;
}

int edpc_load_params(edpc_ctx* c, const float* params, int64_t count) {
  EDPC_CHECK_ARG(c && params, "null argument");
  EDPC_CHECK_ARG(count == c->lay.n_ref, "parameter count mismatch");
  EDPC_CUDA_TRY(cudaSetDevice(c->device));
  const Layout& L = c->lay;
  const int64_t fdm_all = (int64_t)L.B * L.fdm;
  // shared = ref[0, lane_mats) ++ ref[lane_mats + B*fdm, end)
  EDPC_CUDA_TRY(cudaMemcpy(c->W, params, L.ref_lane_mats * 4, cudaMemcpyHostToDevice));
  EDPC_CUDA_TRY(cudaMemcpy(c->W + L.ref_lane_mats, params + L.ref_lane_mats + fdm_all,
                           (L.n_shared - L.ref_lane_mats) * 4, cudaMemcpyHostToDevice));
  EDPC_CUDA_TRY(cudaMemcpy(c->U, params + L.ref_lane_mats + (int64_t)c->lane0 * L.fdm,
                           (int64_t)c->Bl * L.fdm * 4, cudaMemcpyHostToDevice));
  if (c->rt) {  // the tf32-rounded weight shadow starts from the loaded weights
    pdl_launch(k_to_tf32, (unsigned)std::min<int64_t>(cdiv(L.n_shared, 256), 148 * 8), 256, 0, c->st,
               c->W, c->Wt, L.n_shared);
    EDPC_CUDA_TRY(cudaGetLastError());
    EDPC_CUDA_TRY(cudaStreamSynchronize(c->st));
  }
  if (c->h16) {  // the fp16 weight shadow starts from the loaded weights
    pdl_launch(k_to_half, (unsigned)std::min<int64_t>(cdiv(L.n_shared, 256), 148 * 8), 256, 0, c->st, 
        c->W, c->Wh, L.n_shared);
    EDPC_CUDA_TRY(cudaGetLastError());
    EDPC_CUDA_TRY(cudaStreamSynchronize(c->st));
  }
  return EDPC_OK;
}

int edpc_get_params(edpc_ctx* c, float* params, int64_t count) {
  EDPC_CHECK_ARG(c && params, "null argument");
  EDPC_CHECK_ARG(count == c->lay.n_ref, "parameter count mismatch");
  EDPC_CUDA_TRY(cudaSetDevice(c->device));
  EDPC_CUDA_TRY(cudaStreamSynchronize(c->st));
  const Layout& L = c->lay;
  const int64_t fdm_all = (int64_t)L.B * L.fdm;
  EDPC_CUDA_TRY(cudaMemcpy(params, c->W, L.ref_lane_mats * 4, cudaMemcpyDeviceToHost));
  EDPC_CUDA_TRY(cudaMemcpy(params + L.ref_lane_mats + fdm_all, c->W + L.ref_lane_mats,
                           (L.n_shared - L.ref_lane_mats) * 4, cudaMemcpyDeviceToHost));
  EDPC_CUDA_TRY(cudaMemcpy(params + L.ref_lane_mats + (int64_t)c->lane0 * L.fdm, c->U,
                           (int64_t)c->Bl * L.fdm * 4, cudaMemcpyDeviceToHost));
  return EDPC_OK;
}

int edpc_set_input(edpc_ctx* c, const uint8_t* data, int64_t n, int on_device) {
  EDPC_CHECK_ARG(c, "null ctx");
  EDPC_CHECK_ARG(n == c->n, "input length differs from the context's original_len");
  EDPC_CHECK_ARG(n == 0 || data, "null data");
  EDPC_CUDA_TRY(cudaSetDevice(c->device));
  // local lanes [lane0, lane0+Bl) = stream bytes [lane0*L, (lane0+Bl)*L) (zero padded)
  const int64_t start = (int64_t)c->lane0 * c->L;
  const int64_t want = (int64_t)c->Bl * c->L;
  const int64_t have = std::max<int64_t>(0, std::min<int64_t>(want, n - start));
  if (want > have)
    EDPC_CUDA_TRY(cudaMemsetAsync(c->mat + have, 0, want - have, c->st));
  if (have > 0)
    EDPC_CUDA_TRY(cudaMemcpyAsync(c->mat, data + start, have,
                                  on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                                  c->st));
  c->have_input = true;
  return EDPC_OK;
}

int edpc_set_input_columns(edpc_ctx* c, const uint8_t* stream, int64_t n, int64_t col0,
                           int64_t col1) {
  EDPC_CHECK_ARG(c && (stream || n == 0), "null argument");
  EDPC_CHECK_ARG(n == c->n, "input length differs from the context's original_len");
  EDPC_CHECK_ARG(0 <= col0 && col0 <= col1 && col1 <= c->L, "bad column range");
  EDPC_CUDA_TRY(cudaSetDevice(c->device));
  if (!c->have_input) {
    EDPC_CUDA_TRY(cudaMemsetAsync(c->mat, 0, (int64_t)c->Bl * std::max<int64_t>(c->L, 1), c->st));
    EDPC_CUDA_TRY(cudaEventRecord(c->ev_h2d, c->st));
    EDPC_CUDA_TRY(cudaStreamWaitEvent(c->st_h2d, c->ev_h2d, 0));
    c->have_input = true;
  }
  const int64_t w = col1 - col0;
  if (w == 0) return EDPC_OK;
  // copies go on the ingest stream (overlapping the model steps already
  // queued on the main stream); the main stream waits for them before the
  // steps that read these columns.  Rows fully inside the stream go as one
  // strided copy; at most one row is partial.
  int64_t full = 0;
  while (full < c->Bl && ((int64_t)(c->lane0 + full)) * c->L + col1 <= n) ++full;
  if (full)
    EDPC_CUDA_TRY(cudaMemcpy2DAsync(c->mat + col0, c->L, stream + (int64_t)c->lane0 * c->L + col0,
                                    c->L, w, full, cudaMemcpyHostToDevice, c->st_h2d));
  if (full < c->Bl) {
    const int64_t start = (int64_t)(c->lane0 + full) * c->L + col0;
    const int64_t have = std::max<int64_t>(0, std::min<int64_t>(w, n - start));
    if (have)
      EDPC_CUDA_TRY(cudaMemcpyAsync(c->mat + full * c->L + col0, stream + start, have,
                                    cudaMemcpyHostToDevice, c->st_h2d));
  }
  EDPC_CUDA_TRY(cudaEventRecord(c->ev_h2d, c->st_h2d));
  EDPC_CUDA_TRY(cudaStreamWaitEvent(c->st, c->ev_h2d, 0));
  return EDPC_OK;
}

int edpc_set_input_local(edpc_ctx* c, const uint8_t* lanes, int64_t nbytes) {
  EDPC_CHECK_ARG(c && (lanes || nbytes == 0), "null argument");
  const int64_t want = (int64_t)c->Bl * c->L;
  EDPC_CHECK_ARG(nbytes >= 0 && nbytes <= want, "more bytes than the local lanes hold");
  EDPC_CUDA_TRY(cudaSetDevice(c->device));
  if (want > nbytes) EDPC_CUDA_TRY(cudaMemsetAsync(c->mat + nbytes, 0, want - nbytes, c->st));
  if (nbytes) EDPC_CUDA_TRY(cudaMemcpyAsync(c->mat, lanes, nbytes, cudaMemcpyHostToDevice, c->st));
  c->have_input = true;
  return EDPC_OK;
}

int edpc_get_intervals(edpc_ctx* c, int64_t col0, int64_t col1, uint32_t* out) {
  EDPC_CHECK_ARG(c && out, "null argument");
  EDPC_CHECK_ARG(0 <= col0 && col0 <= col1 && col1 <= c->L, "bad column range");
  EDPC_CUDA_TRY(cudaSetDevice(c->device));
  EDPC_CUDA_TRY(cudaMemcpyAsync(out, c->intervals + col0 * c->Bl, (col1 - col0) * c->Bl * 4,
                                cudaMemcpyDeviceToHost, c->st));
  EDPC_CUDA_TRY(cudaStreamSynchronize(c->st));
  return EDPC_OK;
}

int edpc_get_columns(edpc_ctx* c, int64_t col0, int64_t col1, uint8_t* out) {
  EDPC_CHECK_ARG(c && out, "null argument");
  EDPC_CHECK_ARG(0 <= col0 && col0 <= col1 && col1 <= c->L, "bad column range");
  EDPC_CUDA_TRY(cudaSetDevice(c->device));
  if (col1 > col0)
    EDPC_CUDA_TRY(cudaMemcpy2DAsync(out, col1 - col0, c->mat + col0, c->L, col1 - col0, c->Bl,
                                    cudaMemcpyDeviceToHost, c->st));
  EDPC_CUDA_TRY(cudaStreamSynchronize(c->st));
  return EDPC_OK;
}

int edpc_compress_steps(edpc_ctx* c, int64_t i0, int64_t i1) {
  EDPC_CHECK_ARG(c, "null ctx");
  EDPC_CHECK_ARG(c->have_input, "set_input first");
  if (c->finished) {
    set_error("encoder already finished");
    return EDPC_ERR_STATE;
  }
  EDPC_CHECK_ARG(0 <= i0 && i0 <= i1 && i1 <= c->L, "bad column range");
  EDPC_CUDA_TRY(cudaSetDevice(c->device));
  const int T = c->lay.T;
  const int64_t boot = std::min<int64_t>(T, c->L);
  if (i0 < boot) {
    const int64_t a = i0, e = std::min(i1, boot);
    pdl_launch(k_boot_intervals, (unsigned)cdiv((e) * (int64_t)c->Bl, 256), 256, 0, c->st, 
        c->mat, c->L, c->Bl, e, c->intervals);
    EDPC_CUDA_TRY(cudaGetLastError());
    (void)a;
  }
  const int64_t s0 = std::max<int64_t>(i0, T);
  if (s0 < i1) {
    EDPC_TRY(set_step(c, s0, s0 - T + 1));
    EDPC_TRY(run_model_steps(c, i1 - s0, kEncode));
  }
  // DPCA: hand the finished columns to the encoder stream
  c->cols_done = std::max(c->cols_done, i1);
  EDPC_TRY(launch_encoder(c, i1));
  return EDPC_OK;
}

int edpc_compress_finish(edpc_ctx* c, int64_t* bit_lengths, int64_t* total_bytes) {
  EDPC_CHECK_ARG(c && bit_lengths, "null argument");
  if (c->finished) {
    set_error("encoder already finished");
    return EDPC_ERR_STATE;
  }
  EDPC_CUDA_TRY(cudaSetDevice(c->device));
  // a stream is finished after the columns actually produced (normally all L)
  EDPC_TRY(launch_encoder(c, c->cols_done));
  Scope sc(c, kRegEncode, c->st_enc, "encode_finish");
  pdl_launch(k_encode_finish_all, (unsigned)cdiv(c->Sl, 64), 64, 0, c->st_enc, 
      c->enc_state, c->enc_words, c->enc_cap_words, c->Sl);
  EDPC_CUDA_TRY(cudaGetLastError());
  EDPC_CUDA_TRY(cudaStreamSynchronize(c->st_enc));
  EDPC_CUDA_TRY(cudaStreamSynchronize(c->st));
  std::vector<int64_t> es(4 * (size_t)c->Sl);
  EDPC_CUDA_TRY(cudaMemcpy(es.data(), c->enc_state, es.size() * 8, cudaMemcpyDeviceToHost));
  std::vector<int64_t> off(c->Sl + 1, 0);
  for (int s = 0; s < c->Sl; ++s) {
    bit_lengths[s] = es[4 * s + 3];
    off[s + 1] = off[s] + (es[4 * s + 3] + 7) / 8;
  }
  const int64_t tot = off[c->Sl];
  if (total_bytes) *total_bytes = tot;
  // container assembly on the device: the segment payloads packed back to back
  int r = c->alloc(&c->packed, tot + 1);
  if (r != EDPC_OK) return r;
  EDPC_CUDA_TRY(cudaMemcpy(c->pay_off, off.data(), (c->Sl + 1) * 8, cudaMemcpyHostToDevice));
  pdl_launch(k_pack_payloads, (unsigned)c->Sl, 256, 0, c->st_enc, c->enc_words, c->enc_cap_words,
             c->pay_off, c->packed, c->Sl);
  EDPC_CUDA_TRY(cudaGetLastError());
  EDPC_CUDA_TRY(cudaStreamSynchronize(c->st_enc));
  c->packed_bytes = tot;
  c->finished = true;
  return EDPC_OK;
}

int edpc_get_payloads(edpc_ctx* c, uint8_t* out, int64_t cap) {
  EDPC_CHECK_ARG(c && out, "null argument");
  if (!c->finished) {
    set_error("compress_finish first");
    return EDPC_ERR_STATE;
  }
  EDPC_CUDA_TRY(cudaSetDevice(c->device));
  EDPC_CHECK_ARG(c->packed_bytes <= cap, "payload buffer too small");
  if (c->packed_bytes)  // one D2H of the assembled payload area
    EDPC_CUDA_TRY(cudaMemcpy(out, c->packed, c->packed_bytes, cudaMemcpyDeviceToHost));
  return EDPC_OK;
}

int edpc_set_payloads(edpc_ctx* c, const uint8_t* data, const int64_t* bit_lengths) {
  EDPC_CHECK_ARG(c && bit_lengths, "null argument");
  EDPC_CUDA_TRY(cudaSetDevice(c->device));
  std::vector<int64_t> off(c->Sl + 1, 0);
  for (int s = 0; s < c->Sl; ++s) {
    EDPC_CHECK_ARG(bit_lengths[s] >= 0, "negative bit length");
    off[s + 1] = off[s] + (bit_lengths[s] + 7) / 8;
  }
  const int64_t total = off[c->Sl];
  int r = c->alloc(&c->payload, total + 64);
  if (r != EDPC_OK) return r;
  EDPC_CUDA_TRY(cudaMemset(c->payload, 0, total + 64));
  if (total) {
    EDPC_CHECK_ARG(data, "null payload");
    EDPC_CUDA_TRY(cudaMemcpy(c->payload, data, total, cudaMemcpyHostToDevice));
  }
  EDPC_CUDA_TRY(cudaMemcpy(c->pay_off, off.data(), (c->Sl + 1) * 8, cudaMemcpyHostToDevice));
  EDPC_CUDA_TRY(cudaMemcpy(c->bit_len, bit_lengths, c->Sl * 8, cudaMemcpyHostToDevice));
  pdl_launch(k_decoder_init_all, (unsigned)cdiv(c->Sl, 64), 64, 0, c->st, c->dec_state, c->payload,
                                                                 c->pay_off, c->bit_len, c->Sl);
  EDPC_CUDA_TRY(cudaGetLastError());
  EDPC_CUDA_TRY(cudaMemsetAsync(c->mat, 0, (int64_t)c->Bl * std::max<int64_t>(c->L, 1), c->st));
  c->have_payload = true;
  return EDPC_OK;
}

int edpc_decompress_steps(edpc_ctx* c, int64_t i0, int64_t i1) {
  EDPC_CHECK_ARG(c, "null ctx");
  EDPC_CHECK_ARG(c->have_payload, "set_payloads first");
  EDPC_CHECK_ARG(0 <= i0 && i0 <= i1 && i1 <= c->L, "bad column range");
  EDPC_CUDA_TRY(cudaSetDevice(c->device));
  const int T = c->lay.T;
  const int64_t boot = std::min<int64_t>(T, c->L);
  for (int64_t i = i0; i < std::min(i1, boot); ++i) {
    EDPC_TRY(set_step(c, i, 0));
    pdl_launch(k_decode_column, (unsigned)cdiv(c->Sl, 4), 128, 0, c->st, 
        c->mat, c->L, c->si(), c->spl, c->Sl, c->cdf16, true, c->dec_state, c->payload,
        c->pay_off, c->bit_len, c->dec_err);
    EDPC_CUDA_TRY(cudaGetLastError());
  }
  const int64_t s0 = std::max<int64_t>(i0, T);
  if (s0 < i1) {
    EDPC_TRY(set_step(c, s0, s0 - T + 1));
    EDPC_TRY(run_model_steps(c, i1 - s0, kDecode));
  }
  return EDPC_OK;
}

int edpc_get_output(edpc_ctx* c, uint8_t* out, int64_t n_local) {
  EDPC_CHECK_ARG(c && (out || n_local == 0), "null argument");
  EDPC_CUDA_TRY(cudaSetDevice(c->device));
  EDPC_CUDA_TRY(cudaStreamSynchronize(c->st));
  std::vector<int> err(c->Sl);
  EDPC_CUDA_TRY(cudaMemcpy(err.data(), c->dec_err, c->Sl * 4, cudaMemcpyDeviceToHost));
  for (int s = 0; s < c->Sl; ++s)
    if (err[s]) {
      set_error("bitstream exhausted in segment " + std::to_string(c->seg0 + s));
      return EDPC_ERR_CODER;
    }
  EDPC_CHECK_ARG(n_local <= (int64_t)c->Bl * c->L, "output larger than local lanes");
  if (n_local) EDPC_CUDA_TRY(cudaMemcpy(out, c->mat, n_local, cudaMemcpyDeviceToHost));
  return EDPC_OK;
}

int edpc_predict(edpc_ctx* c, const uint8_t* contexts, float* probs) {
  EDPC_CHECK_ARG(c && contexts, "null argument");
  EDPC_CUDA_TRY(cudaSetDevice(c->device));
  const int T = c->lay.T;
  // contexts row b -> scratch[b][0..T)
  EDPC_CUDA_TRY(cudaMemcpy2DAsync(c->scratch, T + 1, contexts, T, T, c->Bl,
                                  cudaMemcpyHostToDevice, c->st));
  EDPC_TRY(set_step(c, T, c->version + 1));
  EDPC_TRY(forward(c, c->seam_src()));
  EDPC_TRY(softmax_quant(c, kProbsOnly, c->seam_src()));
  if (probs)
    EDPC_CUDA_TRY(cudaMemcpyAsync(probs, c->probs, (size_t)c->Bl * 256 * 4,
                                  cudaMemcpyDeviceToHost, c->st));
  EDPC_CUDA_TRY(cudaStreamSynchronize(c->st));
  c->have_cache = true;
  return EDPC_OK;
}

int edpc_train_step(edpc_ctx* c, const uint8_t* targets, float* loss) {
  EDPC_CHECK_ARG(c && targets, "null argument");
  if (!c->have_cache) {
    set_error("stale cache: model was updated since this predict");
    return EDPC_ERR_STATE;
  }
  EDPC_CUDA_TRY(cudaSetDevice(c->device));
  const int T = c->lay.T;
  EDPC_CUDA_TRY(cudaMemcpy2DAsync(c->scratch + T, T + 1, targets, 1, 1, c->Bl,
                                  cudaMemcpyHostToDevice, c->st));
  EDPC_TRY(backward(c, c->seam_src(), c->nll));
  EDPC_TRY(adam_shared(c));
  std::vector<float> nll(c->Bl);
  EDPC_CUDA_TRY(cudaMemcpyAsync(nll.data(), c->nll, c->Bl * 4, cudaMemcpyDeviceToHost, c->st));
  EDPC_CUDA_TRY(cudaStreamSynchronize(c->st));
  double s = 0;
  for (float v : nll) s += v;
  if (loss) *loss = (float)(s / c->lay.B);
  c->version++;
  c->have_cache = false;
  return EDPC_OK;
}

int edpc_last_probs(edpc_ctx* c, float* probs) {
  EDPC_CHECK_ARG(c && probs, "null argument");
  EDPC_CUDA_TRY(cudaSetDevice(c->device));
  EDPC_CUDA_TRY(cudaStreamSynchronize(c->st));
  EDPC_CUDA_TRY(cudaMemcpy(probs, c->probs, (size_t)c->Bl * 256 * 4, cudaMemcpyDeviceToHost));
  return EDPC_OK;
}

int edpc_step_phase(edpc_ctx* c, int64_t i, int32_t phase, int32_t decompress) {
  EDPC_CHECK_ARG(c, "null ctx");
  EDPC_CHECK_ARG(i >= c->lay.T && i < c->L, "step index out of range");
  EDPC_CUDA_TRY(cudaSetDevice(c->device));
  ByteCols src = c->lanes_src();
  if (phase == 0) {
    EDPC_TRY(set_step(c, i, i - c->lay.T + 1));
    EDPC_TRY(forward(c, src));
    EDPC_TRY(softmax_quant(c, decompress ? kDecode : kEncode, src));
    if (decompress) {
      pdl_launch(k_decode_column, (unsigned)cdiv(c->Sl, 4), 128, 0, c->st, 
          c->mat, c->L, c->si(), c->spl, c->Sl, c->cdf16, false, c->dec_state, c->payload,
          c->pay_off, c->bit_len, c->dec_err);
      EDPC_CUDA_TRY(cudaGetLastError());
    }
    EDPC_TRY(backward(c, src, nullptr, !decompress));
    EDPC_TRY(group_tree(c));
    if (!decompress) c->cols_done = std::max(c->cols_done, i + 1);
    return EDPC_OK;
  }
  EDPC_CHECK_ARG(phase == 1, "phase must be 0 or 1");
  EDPC_TRY(exchange_slices(c));
  EDPC_TRY(adam_shared(c));
  EDPC_TRY(exchange_weights(c));
  return EDPC_OK;
}

int edpc_encode_pending(edpc_ctx* c, int64_t upto) {
  EDPC_CHECK_ARG(c, "null ctx");
  EDPC_CHECK_ARG(upto <= c->cols_done, "columns not produced yet");
  EDPC_CUDA_TRY(cudaSetDevice(c->device));
  return launch_encoder(c, upto);
}

int edpc_partials_copy(edpc_ctx* c, int32_t g0, int32_t ng, float* host, int32_t to_device) {
  EDPC_CHECK_ARG(c && host && g0 >= 0 && ng >= 0 && g0 + ng <= kNumGroups, "bad arguments");
  EDPC_CUDA_TRY(cudaSetDevice(c->device));
  float* dev = c->Gp + (size_t)g0 * c->lay.n_shared;
  const size_t bytes = (size_t)ng * c->lay.n_shared * 4;
  if (to_device)
    EDPC_CUDA_TRY(cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, c->st));
  else
    EDPC_CUDA_TRY(cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, c->st));
  EDPC_CUDA_TRY(cudaStreamSynchronize(c->st));
  return EDPC_OK;
}

// Peer copy src -> dst of `bytes` on dst's stream, ordered after src's queued
// work; src's later work is ordered after the copy.
static int pull_ordered(edpc_ctx* dst, edpc_ctx* src, void* to, const void* from, size_t bytes) {
  EDPC_CUDA_TRY(cudaSetDevice(src->device));
  EDPC_CUDA_TRY(cudaEventRecord(src->ev, src->st));
  EDPC_CUDA_TRY(cudaSetDevice(dst->device));
  EDPC_CUDA_TRY(cudaStreamWaitEvent(dst->st, src->ev, 0));
  EDPC_CUDA_TRY(cudaMemcpyPeerAsync(to, dst->device, from, src->device, bytes, dst->st));
  EDPC_CUDA_TRY(cudaEventRecord(dst->ev, dst->st));
  EDPC_CUDA_TRY(cudaSetDevice(src->device));
  EDPC_CUDA_TRY(cudaStreamWaitEvent(src->st, dst->ev, 0));
  return EDPC_OK;
}

static bool same_shard_set(const edpc_ctx* a, const edpc_ctx* b) {
  return a->lay.n_shared == b->lay.n_shared && a->g_count == b->g_count && a->h16 == b->h16 &&
         a->rt == b->rt;
}

// Sharded-optimizer step 2 without NCCL (dist.ShardSet): dst <- src's subtree
// sum of dst's owned parameter slice, into slot src->g_first (device to
// device; a peer copy over NVLink when the contexts sit on different GPUs).
int edpc_partials_pull(edpc_ctx* dst, edpc_ctx* src) {
  EDPC_CHECK_ARG(dst && src && same_shard_set(dst, src), "bad contexts");
  if (src == dst || shard_count(dst) < 2) return EDPC_OK;
  int64_t off, len;
  shard_range(dst, shard_rank(dst), &off, &len);
  if (len <= 0) return EDPC_OK;
  const size_t at = (size_t)src->g_first * src->lay.n_shared + (size_t)off;
  return pull_ordered(dst, src, dst->Gp + at, src->Gp + at, (size_t)len * 4);
}

// Sharded-optimizer step 4 without NCCL: dst <- src's owned slice of the
// updated weights (fp32 and the fp16 shadow).
int edpc_weights_pull(edpc_ctx* dst, edpc_ctx* src) {
  EDPC_CHECK_ARG(dst && src && same_shard_set(dst, src), "bad contexts");
  if (src == dst || shard_count(src) < 2) return EDPC_OK;
  int64_t off, len;
  shard_range(src, shard_rank(src), &off, &len);
  if (len <= 0) return EDPC_OK;
  EDPC_TRY(pull_ordered(dst, src, dst->W + off, src->W + off, (size_t)len * 4));
  if (src->h16) EDPC_TRY(pull_ordered(dst, src, dst->Wh + off, src->Wh + off, (size_t)len * 2));
  if (src->rt) EDPC_TRY(pull_ordered(dst, src, dst->Wt + off, src->Wt + off, (size_t)len * 4));
  return EDPC_OK;
}

int edpc_shard_range(edpc_ctx* c, int64_t* off, int64_t* len) {
  EDPC_CHECK_ARG(c && off && len, "null argument");
  shard_range(c, shard_rank(c), off, len);
  return EDPC_OK;
}

int edpc_ctx_groups(edpc_ctx* c, int32_t* g_first, int32_t* g_count) {
  EDPC_CHECK_ARG(c && g_first && g_count, "null argument");
  *g_first = c->g_first;
  *g_count = c->g_count;
  return EDPC_OK;
}

int edpc_nccl_unique_id(uint8_t* out, int32_t cap) {
  EDPC_CHECK_ARG(out && cap >= (int32_t)sizeof(ncclUniqueId), "buffer too small");
  if (!nccl().ok) {
    set_error("libnccl.so.2 not loadable");
    return EDPC_ERR_CUDA;
  }
  ncclUniqueId id;
  ncclResult_t r = nccl().getUniqueId(&id);
  if (r != ncclSuccess) {
    set_error(std::string("ncclGetUniqueId: ") + nccl().getErrorString(r));
    return EDPC_ERR_CUDA;
  }
  memcpy(out, &id, sizeof(id));
  return EDPC_OK;
}

// Joins the context to an NCCL communicator (collective: every rank calls it
// concurrently with the same id).  Requires whole, equal lane-group shares.
int edpc_ctx_set_comm(edpc_ctx* c, const uint8_t* id, int32_t nranks, int32_t rank) {
  EDPC_CHECK_ARG(c && id, "null argument");
  EDPC_CHECK_ARG(nranks >= 1 && rank >= 0 && rank < nranks, "bad rank");
  EDPC_CHECK_ARG(kNumGroups % nranks == 0 && c->lay.B % kNumGroups == 0,
                 "multi-GPU needs lanes % 8 == 0 and a GPU count dividing 8");
  EDPC_CHECK_ARG(c->g_count == kNumGroups / nranks && c->g_first == rank * c->g_count &&
                     c->lane0 == group_begin(c->g_first, c->lay.B) &&
                     c->Bl == group_begin(c->g_first + c->g_count, c->lay.B) - c->lane0,
                 "rank must own lane groups [rank*8/G, (rank+1)*8/G) exactly");
  EDPC_CUDA_TRY(cudaSetDevice(c->device));
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  if (!nccl().ok) {
    set_error("libnccl.so.2 not loadable");
    return EDPC_ERR_CUDA;
  }
  ncclComm_t comm;
  ncclResult_t r = nccl().commInitRank(&comm, nranks, uid, rank);
  if (r != ncclSuccess) {
    set_error(std::string("ncclCommInitRank: ") + nccl().getErrorString(r));
    return EDPC_ERR_CUDA;
  }
  if (c->comm) nccl().commDestroy(c->comm);
  c->comm = comm;
  c->nranks = nranks;
  c->rank = rank;
  c->wfuse = false;  // the slice exchange needs the group partials
  c->wsub = false;
  for (auto& g : c->graph)  // captured steps must include the collective
    if (g) {
      cudaGraphExecDestroy(g);
      g = nullptr;
    }
  return EDPC_OK;
}

int edpc_grad_partials(edpc_ctx* c, float** dev_ptr, int64_t* n_shared) {
  EDPC_CHECK_ARG(c && dev_ptr && n_shared, "null argument");
  *dev_ptr = c->Gp;
  *n_shared = c->lay.n_shared;
  return EDPC_OK;
}

int edpc_prof(edpc_ctx* c, int enable) {
  EDPC_CHECK_ARG(c, "null ctx");
  EDPC_CUDA_TRY(cudaSetDevice(c->device));
  cudaStreamSynchronize(c->st);
  cudaStreamSynchronize(c->st_aux);
  cudaStreamSynchronize(c->st_enc);
  c->prof.reset();
  c->prof.on = enable != 0;
  return EDPC_OK;
}

int edpc_prof_read(edpc_ctx* c, int32_t region, double* ms, int64_t* count) {
  EDPC_CHECK_ARG(c && ms && count, "null argument");
  EDPC_CHECK_ARG(region >= -1 && region < kNumRegions, "bad region");
  EDPC_CUDA_TRY(cudaSetDevice(c->device));
  cudaStreamSynchronize(c->st);
  cudaStreamSynchronize(c->st_aux);
  cudaStreamSynchronize(c->st_enc);
  c->prof.flush();
  if (region < 0) {
    *ms = 0;
    *count = c->prof.launches;
  } else {
    *ms = c->prof.ms[region];
    *count = c->prof.n[region];
  }
  return EDPC_OK;
}

int edpc_timer(edpc_ctx* c, int32_t op, double* ms) {
  EDPC_CHECK_ARG(c, "null ctx");
  EDPC_CUDA_TRY(cudaSetDevice(c->device));
  if (!c->t0) {
    EDPC_CUDA_TRY(cudaEventCreate(&c->t0));
    EDPC_CUDA_TRY(cudaEventCreate(&c->t1));
    EDPC_CUDA_TRY(cudaEventCreateWithFlags(&c->tj, cudaEventDisableTiming));
  }
  if (op == 0) {  // start: after everything queued on both streams so far
    EDPC_CUDA_TRY(cudaEventRecord(c->tj, c->st_enc));
    EDPC_CUDA_TRY(cudaStreamWaitEvent(c->st, c->tj, 0));
    EDPC_CUDA_TRY(cudaEventRecord(c->t0, c->st));
  } else if (op == 1) {  // stop: joins the encoder stream first (DPCA stage B)
    EDPC_CUDA_TRY(cudaEventRecord(c->tj, c->st_enc));
    EDPC_CUDA_TRY(cudaStreamWaitEvent(c->st, c->tj, 0));
    EDPC_CUDA_TRY(cudaEventRecord(c->t1, c->st));
  } else {
    EDPC_CHECK_ARG(ms, "null ms");
    EDPC_CUDA_TRY(cudaEventSynchronize(c->t1));
    float t = 0.f;
    EDPC_CUDA_TRY(cudaEventElapsedTime(&t, c->t0, c->t1));
    *ms = t;
  }
  return EDPC_OK;
}

// Standalone GEMM through the tcgen05 path (tests): C[M][N] = A . B with A
// given [M][K] (a_mn = 0) or [K][M] (a_mn = 1) and B [N][K] (b_mn = 0) or
// [K][N] (b_mn = 1), all row-major fp32 host arrays.
int edpc_debug_gemm(int32_t M, int32_t N, int32_t K, int32_t a_mn, int32_t b_mn, const float* A,
                    const float* B, float* C, int32_t dbg) {
  EDPC_CHECK_ARG(A && B && C && M > 0 && N > 0 && K > 0, "bad arguments");
  EDPC_CHECK_ARG(tc_shape_ok(N, K), "shape not supported by the tcgen05 path");
  float *dA, *dB, *dC;
  EDPC_CUDA_TRY(cudaMalloc(&dA, (size_t)M * K * 4));
  EDPC_CUDA_TRY(cudaMalloc(&dB, (size_t)N * K * 4));
  EDPC_CUDA_TRY(cudaMalloc(&dC, (size_t)M * N * 4));
  EDPC_CUDA_TRY(cudaMemcpy(dA, A, (size_t)M * K * 4, cudaMemcpyHostToDevice));
  EDPC_CUDA_TRY(cudaMemcpy(dB, B, (size_t)N * K * 4, cudaMemcpyHostToDevice));
  EDPC_CUDA_TRY(cudaMemset(dC, 0, (size_t)M * N * 4));
  TcShape s{M, N, K, 1, 1, kBatchNone, kBatchNone, 0, 1, 0, 0, 0, dbg};
  TcOperand a{dA, a_mn ? M : K, 0, 1}, b{dB, b_mn ? N : K, 0, 1};
  EpiStore e{dC, N};
  int st;
  if (!a_mn && !b_mn) st = tc_gemm<false, false>(s, a, b, e, 0);
  else if (!a_mn && b_mn) st = tc_gemm<false, true>(s, a, b, e, 0);
  else if (a_mn && !b_mn) st = tc_gemm<true, false>(s, a, b, e, 0);
  else st = tc_gemm<true, true>(s, a, b, e, 0);
  cudaError_t ce = cudaDeviceSynchronize();
  if (st == EDPC_OK && ce == cudaSuccess)
    ce = cudaMemcpy(C, dC, (size_t)M * N * 4, cudaMemcpyDeviceToHost);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dC);
  if (st != EDPC_OK) return st;
  EDPC_CUDA_TRY(ce);
  return EDPC_OK;
}

__global__ void k_fill_rand(float* p, int64_t n, uint32_t seed) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u ^ seed;
    h ^= h >> 15;
    h *= 2246822519u;
    h ^= h >> 13;
    p[i] = (float)(h & 0xffff) / 65536.0f - 0.5f;
  }
}

// fp16-operand GEMM of host matrices (tests): A, B as IEEE half bits;
// lbo/sbo override the MN-major descriptor strides (0 = default).
int edpc_debug_gemm_h(int32_t M, int32_t N, int32_t K, int32_t a_mn, int32_t b_mn,
                      const uint16_t* A, const uint16_t* B, float* C, int32_t lbo, int32_t sbo) {
  EDPC_CHECK_ARG(A && B && C && M > 0 && N > 0 && K > 0, "bad arguments");
  EDPC_CHECK_ARG(N % 64 == 0 && K % tc_bk<true>() == 0 && (N <= 256 || N % 256 == 0),
                 "shape not supported by the fp16 tcgen05 path");
  uint16_t *dA, *dB;
  float* dC;
  EDPC_CUDA_TRY(cudaMalloc(&dA, (size_t)M * K * 2));
  EDPC_CUDA_TRY(cudaMalloc(&dB, (size_t)N * K * 2));
  EDPC_CUDA_TRY(cudaMalloc(&dC, (size_t)M * N * 4));
  EDPC_CUDA_TRY(cudaMemcpy(dA, A, (size_t)M * K * 2, cudaMemcpyHostToDevice));
  EDPC_CUDA_TRY(cudaMemcpy(dB, B, (size_t)N * K * 2, cudaMemcpyHostToDevice));
  EDPC_CUDA_TRY(cudaMemset(dC, 0, (size_t)M * N * 4));
  TcShape s{M, N, K, 1, 1, kBatchNone, kBatchNone, 0, 1, 0, 0, 0};
  s.mn_lbo = lbo;
  s.mn_sbo = sbo;
  TcOperand a{dA, a_mn ? M : K, 0, 1}, b{dB, b_mn ? N : K, 0, 1};
  EpiStore e{dC, N};
  int st;
  if (!a_mn && !b_mn) st = tc_gemm<false, false, true>(s, a, b, e, 0);
  else if (!a_mn && b_mn) st = tc_gemm<false, true, true>(s, a, b, e, 0);
  else if (a_mn && !b_mn) st = tc_gemm<true, false, true>(s, a, b, e, 0);
  else st = tc_gemm<true, true, true>(s, a, b, e, 0);
  cudaError_t ce = cudaDeviceSynchronize();
  if (st == EDPC_OK && ce == cudaSuccess)
    ce = cudaMemcpy(C, dC, (size_t)M * N * 4, cudaMemcpyDeviceToHost);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dC);
  if (st != EDPC_OK) return st;
  EDPC_CUDA_TRY(ce);
  return EDPC_OK;
}

// Microbenchmark of the bare tcgen05 GEMM (store-only epilogue) on device
// operands: average ms over iters launches (CUDA events).  kmode 2 splits K.
int edpc_bench_gemm(int32_t M, int32_t N, int32_t K, int32_t a_mn, int32_t b_mn, int32_t nsplit,
                    int32_t iters, double* ms) {
  EDPC_CHECK_ARG(ms && M > 0 && N > 0 && K > 0 && iters > 0 && nsplit >= 1, "bad arguments");
  EDPC_CHECK_ARG(tc_shape_ok(N, K / nsplit), "shape not supported by the tcgen05 path");
  float *dA, *dB, *dC;
  EDPC_CUDA_TRY(cudaMalloc(&dA, (size_t)M * K * 4));
  EDPC_CUDA_TRY(cudaMalloc(&dB, (size_t)N * K * 4));
  EDPC_CUDA_TRY(cudaMalloc(&dC, (size_t)nsplit * M * N * 4));
  k_fill_rand<<<1024, 256>>>(dA, (int64_t)M * K, 1u);
  k_fill_rand<<<1024, 256>>>(dB, (int64_t)N * K, 2u);
  TcShape s{M, N, K, 1, 1, kBatchNone, kBatchNone, nsplit > 1 ? 2 : 0, nsplit, 0, 0, 0};
  TcOperand a{dA, a_mn ? M : K, 0, 1}, b{dB, b_mn ? N : K, 0, 1};
  if (const char* d = getenv("EDPC_GEMM_DBG")) s.dbg = atoi(d);
  EpiSplit e{dC, N, (int64_t)M * N};
  const char* hf = getenv("EDPC_GEMM_F16");  // fp16 operands (timing only: the fp32
  const bool h = hf && hf[0] == '1';          // random bits are read as halves)
  auto run = [&]() {
    if (h) {
      if (!a_mn && !b_mn) return tc_gemm<false, false, true>(s, a, b, e, 0);
      if (!a_mn && b_mn) return tc_gemm<false, true, true>(s, a, b, e, 0);
      if (a_mn && !b_mn) return tc_gemm<true, false, true>(s, a, b, e, 0);
      return tc_gemm<true, true, true>(s, a, b, e, 0);
    }
    if (!a_mn && !b_mn) return tc_gemm<false, false>(s, a, b, e, 0);
    if (!a_mn && b_mn) return tc_gemm<false, true>(s, a, b, e, 0);
    if (a_mn && !b_mn) return tc_gemm<true, false>(s, a, b, e, 0);
    return tc_gemm<true, true>(s, a, b, e, 0);
  };
  int st = run();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, 0);
  for (int i = 0; i < iters && st == EDPC_OK; ++i) st = run();
  cudaEventRecord(e1, 0);
  cudaError_t ce = cudaEventSynchronize(e1);
  float t = 0.f;
  cudaEventElapsedTime(&t, e0, e1);
  *ms = t / iters;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dC);
  if (st != EDPC_OK) return st;
  EDPC_CUDA_TRY(ce);
  return EDPC_OK;
}

int edpc_debug_read(edpc_ctx* c, int32_t which, float* out, int64_t count) {
  EDPC_CHECK_ARG(c && out, "null argument");
  EDPC_CUDA_TRY(cudaSetDevice(c->device));
  EDPC_CUDA_TRY(cudaStreamSynchronize(c->st));
  const Layout& L = c->lay;
  const int64_t Bl = c->Bl;
  const float* src = nullptr;
  int64_t n = 0;
  switch (which) {
    case 0: src = c->Gp; n = (int64_t)kNumGroups * L.n_shared; break;
    case 1: src = c->probs; n = Bl * 256; break;
    case 2: src = c->x_local; n = Bl * L.F; break;
    case 3: src = c->x_lte; n = Bl * L.F; break;
    case 4: src = c->x_global; n = Bl * L.F; break;
    case 5: src = c->l_H; n = (int64_t)L.K * Bl * L.HL; break;
    case 6: src = c->g_H; n = (int64_t)L.K * Bl * L.HG; break;
    case 7: src = c->g_emb; n = Bl * L.F; break;
    case 8: src = c->logits; n = Bl * 256; break;
    case 9: src = c->Um; n = Bl * L.fdm; break;   // per-lane FDM Adam m
    case 10: src = c->M; n = L.n_shared; break;   // shared Adam m
    case 11: src = c->V; n = L.n_shared; break;   // shared Adam v
    case 12: src = c->U; n = Bl * L.fdm; break;   // per-lane FDM U
    default: EDPC_CHECK_ARG(false, "unknown debug buffer");
  }
  EDPC_CHECK_ARG(count == n, "debug buffer size mismatch (expected " + std::to_string(n) + ")");
  if (c->h16 && (which == 5 || which == 6)) {  // D_z stored as fp16 on that path
    std::vector<__half> h((size_t)n);
    EDPC_CUDA_TRY(cudaMemcpy(h.data(), src, n * 2, cudaMemcpyDeviceToHost));
    for (int64_t e = 0; e < n; ++e) out[e] = __half2float(h[(size_t)e]);
    return EDPC_OK;
  }
  EDPC_CUDA_TRY(cudaMemcpy(out, src, n * 4, cudaMemcpyDeviceToHost));
  if (which == 0) {  // partials are kept in gradient-scale units (k_dlogits)
    const float inv = ldexpf(1.0f, -c->gs_log2);
    for (int64_t e = 0; e < n; ++e) out[e] *= inv;
  }
  return EDPC_OK;
}

// The shared-parameter Adam kernel (k_adam_shared, one leaf) on host arrays:
// `steps` updates of w0 by grads[t][n], t = 1..steps (`_kernels.py:18-32`,
// the reference's adam_update over a flat buffer).  Tests pin it against the
// reference-generated trajectory (tests/golden/adam.npz).
int edpc_debug_adam(const float* w0, const float* grads, int64_t n, int32_t steps, double lr,
                    double beta1, double beta2, double eps, float* w_out, float* m_out,
                    float* v_out) {
  EDPC_CHECK_ARG(w0 && grads && w_out && m_out && v_out && n > 0 && steps >= 0, "bad arguments");
  float *W, *M, *V, *P;
  int64_t* d_t;
  EDPC_CUDA_TRY(cudaMalloc(&W, n * 4));
  EDPC_CUDA_TRY(cudaMalloc(&M, n * 4));
  EDPC_CUDA_TRY(cudaMalloc(&V, n * 4));
  EDPC_CUDA_TRY(cudaMalloc(&P, n * 4));
  EDPC_CUDA_TRY(cudaMalloc(&d_t, 8));
  EDPC_CUDA_TRY(cudaMemcpy(W, w0, n * 4, cudaMemcpyHostToDevice));
  EDPC_CUDA_TRY(cudaMemset(M, 0, n * 4));
  EDPC_CUDA_TRY(cudaMemset(V, 0, n * 4));
  AdamConsts a{};
  a.lr = (float)lr;
  a.b1 = (float)beta1;
  a.b2 = (float)beta2;
  a.k1 = (float)(1.0 - beta1);
  a.k2 = (float)(1.0 - beta2);
  a.eps = (float)eps;
  cudaError_t e = cudaSuccess;
  for (int32_t t = 1; t <= steps && e == cudaSuccess; ++t) {
    const int64_t tt = t;
    e = cudaMemcpy(d_t, &tt, 8, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(P, grads + (t - 1) * n, n * 4, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
      k_adam_shared<1><<<(unsigned)std::min<int64_t>(cdiv(n, 256), 1184), 256>>>(
          W, M, V, P, n, n, StepIdx{d_t, d_t, 0}, a, beta1, beta2, 1.0f, nullptr, nullptr);
      e = cudaDeviceSynchronize();
    }
  }
  if (e == cudaSuccess) e = cudaMemcpy(w_out, W, n * 4, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(m_out, M, n * 4, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(v_out, V, n * 4, cudaMemcpyDeviceToHost);
  cudaFree(W);
  cudaFree(M);
  cudaFree(V);
  cudaFree(P);
  cudaFree(d_t);
  EDPC_CUDA_TRY(e);
  return EDPC_OK;
}

// Debug: with fused weight-gradient/Adam kernels the 8 lane-group partials
// are never materialised; keep = 1 makes those kernels also write the reduced
// gradient (gradient-scale units) into partial slot 0, slots 1..7 zero, so
// edpc_debug_read(0) keeps its meaning (tree of the 8 slots = the gradient).
int edpc_debug_keep_grads(edpc_ctx* c, int32_t keep) {
  EDPC_CHECK_ARG(c, "null ctx");
  EDPC_CUDA_TRY(cudaSetDevice(c->device));
  EDPC_CUDA_TRY(cudaStreamSynchronize(c->st));
  c->keep_grads = keep != 0;
  EDPC_CUDA_TRY(cudaMemset(c->Gp, 0, (size_t)kNumGroups * c->lay.n_shared * 4));
  for (auto& g : c->graph)  // captured launches carry the pointer
    if (g) {
      cudaGraphExecDestroy(g);
      g = nullptr;
    }
  return EDPC_OK;
}

int edpc_trim_pool(int32_t device) {
  EDPC_CUDA_TRY(cudaSetDevice(device));
  cudaMemPool_t pool;
  EDPC_CUDA_TRY(cudaDeviceGetDefaultMemPool(&pool, device));
  EDPC_CUDA_TRY(cudaDeviceSynchronize());
  EDPC_CUDA_TRY(cudaMemPoolTrimTo(pool, 0));
  return EDPC_OK;
}

int edpc_sync(edpc_ctx* c) {
  EDPC_CHECK_ARG(c, "null ctx");
  EDPC_CUDA_TRY(cudaSetDevice(c->device));
  EDPC_CUDA_TRY(cudaStreamSynchronize(c->st_aux));
  EDPC_CUDA_TRY(cudaStreamSynchronize(c->st));
  EDPC_CUDA_TRY(cudaStreamSynchronize(c->st_enc));
  return EDPC_OK;
}

}  // extern "C"
