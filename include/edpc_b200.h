/*
 * edpc_b200.h -- C ABI of the B200-native EDPC compression hot path.
 *
 * Plain C: opaque handles, raw pointers, sizes and int status codes; no torch
 * or C++ types cross this boundary.  Every call returns EDPC_OK (0) or a
 * nonzero edpc_status; edpc_last_error() gives the thread's last message.
 *
 * Each entry point replaces one reference interface (pkg/src/edpc/...):
 *
 *   edpc_quantize_rows     <- coder.py:83-106  quantize_rows / _quantize_kernel :58-80
 *   edpc_encode_rows       <- coder.py:264-271 ArithmeticEncoder.encode_rows / _encode_kernel :126-165
 *   edpc_encode_finish     <- coder.py:290-306 ArithmeticEncoder.finish
 *   edpc_decoder_init      <- coder.py:317-333 ArithmeticDecoder.__init__ (code-register priming)
 *   edpc_decode_rows       <- coder.py:335-340 ArithmeticDecoder.decode_rows / _decode_kernel :177-229
 *   edpc_ctx_create        <- pipeline.py:120-137 geometry + EdpcModel(cfg) construction (model.py:187-199)
 *   edpc_load_params       <- model.py:201-221 flat parameter buffers (parameters() order)
 *   edpc_get_params        <- model.py:294-300 state_checksum's byte source
 *   edpc_set_input         <- pipeline.py:44-56 split_lanes (on device)
 *   edpc_compress_steps    <- pipeline.py:137,194-211 bootstrap + predict/encode/train loop
 *   edpc_compress_finish   <- pipeline.py:221-227 ArithmeticEncoder.finish per segment
 *   edpc_set_payloads      <- pipeline.py:258-261 ArithmeticDecoder per segment
 *   edpc_decompress_steps  <- pipeline.py:261,278-290 bootstrap + predict/decode/train loop
 *   edpc_get_output        <- pipeline.py:295 join_lanes
 *   edpc_predict           <- model.py:241-263 EdpcModel.predict
 *   edpc_train_step        <- model.py:265-281 EdpcModel.train_step
 *
 * Threading: calls on one edpc_ctx must be serialised by the caller (the
 * reference's "one owner thread" rule).  Distinct contexts may
 * be driven from distinct host threads.
 */
#ifndef EDPC_B200_H
#define EDPC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EDPC_ABI_VERSION 1

typedef enum {
  EDPC_OK = 0,
  EDPC_ERR_INVALID = 1,   /* bad argument / geometry (reference: ValueError) */
  EDPC_ERR_CUDA = 2,      /* CUDA runtime failure or no usable device */
  EDPC_ERR_CODER = 3,     /* bitstream exhausted (reference: CoderError) */
  EDPC_ERR_STATE = 4,     /* call out of order: stale cache, finished coder */
  EDPC_ERR_NOMEM = 5      /* device allocation failed */
} edpc_status;

typedef struct {
  int32_t context_len;
  int32_t embed_dim;
  int32_t hidden_local;
  int32_t hidden_global;
  int32_t lte_ratio;
  int32_t branches;
  int32_t lanes;          /* global lane count B (the container's) */
  int32_t _pad;
  double lr;
  double beta1;
  double beta2;
  double adam_eps;
  uint64_t seed;
} edpc_config;

typedef struct edpc_ctx edpc_ctx;

const char* edpc_last_error(void);
int edpc_abi_version(void);
int edpc_device_count(int* count);
/* 1 if the library was built with the tcgen05 (sm_100a) GEMM path compiled in */
int edpc_has_tcgen05(void);

/* ---------------------------------------------------------------- coder parity
 * Stateless w.r.t. the library: the caller owns the coder registers.
 * dtype: 0 = float32 rows, 1 = float64 rows.  cums rows are 257 x uint32. */
int edpc_quantize_rows(int device, const void* probs, int64_t n, int dtype, uint32_t* cums);

/* enc_state = {low, high, pending, bitpos}; buf holds cap bytes, zero beyond bitpos. */
int edpc_encode_rows(int device, int64_t* enc_state, uint8_t* buf, int64_t cap,
                     const uint32_t* cums, const int32_t* symbols, int64_t n);
int edpc_encode_finish(int device, int64_t* enc_state, uint8_t* buf, int64_t cap,
                       int64_t* bit_length);

/* dec_state = {low, high, code, bitpos}; decoded symbols into out (int32);
 * *done = rows decoded (< n means exhausted: EDPC_ERR_CODER). */
int edpc_decoder_init(int device, int64_t* dec_state, const uint8_t* data, int64_t nbytes,
                      int64_t bit_length);
int edpc_decode_rows(int device, int64_t* dec_state, const uint8_t* data, int64_t nbytes,
                     int64_t bit_length, const uint32_t* cums, int64_t n, int32_t* out,
                     int64_t* done);

/* ------------------------------------------------------------ context (stream)
 * One context = one container being (de)compressed on one device.
 * lane_begin/lane_count select this device's contiguous share of the B lanes
 * (whole segments); single-GPU callers pass 0 and cfg->lanes.
 * original_len is the full stream length n (L = ceil(n / B)). */
int edpc_ctx_create(const edpc_config* cfg, int32_t segments, int64_t original_len,
                    int32_t device, int32_t lane_begin, int32_t lane_count, edpc_ctx** out);
/* Same, with the numerics forced: numerics = -1 picks the policy default (a
 * function of the config); otherwise the EDPC_NUM_* flags below, as recorded
 * in a container header (the decoder replays the encoder's numerics).  Flags
 * the config / build cannot run are refused with EDPC_ERR_INVALID. */
int edpc_ctx_create_ex(const edpc_config* cfg, int32_t segments, int64_t original_len,
                       int32_t device, int32_t lane_begin, int32_t lane_count, int32_t numerics,
                       edpc_ctx** out);
int edpc_ctx_destroy(edpc_ctx* ctx);
/* Numerics the context runs (part of the format, stored in the container's
 * version byte): */
#define EDPC_NUM_TCGEN05 1   /* tcgen05 tensor-core GEMMs (tf32 operands)          */
#define EDPC_NUM_FP16 2      /* fp16 operands for the MBRB branch / out-projection */
#define EDPC_NUM_LTE_FUSED 4 /* fused LTE forward kernel (mma.sync tf32, rna)      */
#define EDPC_NUM_RND_TF32 8  /* tf32 GEMM operands rounded to nearest (a rounded   */
                             /* weight shadow; producers store rounded operands)   */
int edpc_ctx_numerics(edpc_ctx* ctx, int32_t* flags);
int edpc_ctx_info(edpc_ctx* ctx, int64_t* lane_len, int64_t* n_params, int64_t* n_shared);

/* fp32 parameters in the reference parameters() order (model.py:237-239),
 * full lane_mats for all B lanes (the context keeps its own lanes' slice). */
int edpc_load_params(edpc_ctx* ctx, const float* params, int64_t count);
int edpc_get_params(edpc_ctx* ctx, float* params, int64_t count);

/* compress side: stream bytes (host or device pointer) -> device lane matrix */
int edpc_set_input(edpc_ctx* ctx, const uint8_t* data, int64_t n, int on_device);
/* streaming ingestion: lane columns [col0, col1) of the local lanes copied
 * from the host stream (pitch L; zero padding past n) -- pipeline.py:44-56
 * done column-block by column-block so H2D overlaps the model steps */
int edpc_set_input_columns(edpc_ctx* ctx, const uint8_t* stream, int64_t n, int64_t col0,
                           int64_t col1);
/* the local lanes' bytes only ([lane_count][L] row-major, zero padded past nbytes) */
int edpc_set_input_local(edpc_ctx* ctx, const uint8_t* lanes, int64_t nbytes);
/* coded intervals (cum_lo | freq << 16) of lane columns [col0, col1), [col][lane] */
int edpc_get_intervals(edpc_ctx* ctx, int64_t col0, int64_t col1, uint32_t* out);
/* lane-matrix columns [col0, col1) as [lane][col] (decoded bytes on the decode side) */
int edpc_get_columns(edpc_ctx* ctx, int64_t col0, int64_t col1, uint8_t* out);
/* runs lane columns [i0, i1) (bootstrap for i < context_len, model steps after) */
int edpc_compress_steps(edpc_ctx* ctx, int64_t i0, int64_t i1);
/* finishes every local segment; bit_lengths[S_local], payload bytes total */
int edpc_compress_finish(edpc_ctx* ctx, int64_t* bit_lengths, int64_t* total_bytes);
/* concatenated local payloads (ceil(bits/8) bytes each, in segment order) */
int edpc_get_payloads(edpc_ctx* ctx, uint8_t* out, int64_t cap);

/* decompress side */
int edpc_set_payloads(edpc_ctx* ctx, const uint8_t* data, const int64_t* bit_lengths);
int edpc_decompress_steps(edpc_ctx* ctx, int64_t i0, int64_t i1);
int edpc_get_output(edpc_ctx* ctx, uint8_t* out, int64_t n_local);

/* model-level seam: one predict / train_step on caller contexts (host memory).
 * contexts: lane_count x context_len bytes; probs: lane_count x 256 fp32
 * (may be NULL); targets: lane_count bytes; loss: mean NLL in nats over the
 * local lanes' share (sum_local / B). */
int edpc_predict(edpc_ctx* ctx, const uint8_t* contexts, float* probs);
int edpc_train_step(edpc_ctx* ctx, const uint8_t* targets, float* loss);
/* probs of the last model step run by compress/decompress_steps (debug taps) */
int edpc_last_probs(edpc_ctx* ctx, float* probs);

/* --------------------------------------------------- multi-GPU step phases
 * Replaces the reference's single shared-model update (model.py:265-281,
 * _adam_all model.py:223-235) when the lanes of one container are sharded
 * over G contexts (G divides 8, rank r owns lane groups
 * [r*8/G, (r+1)*8/G)).  Sharded optimizer, per model step:
 *   phase 0: forward, coder, backward, per-lane FDM update; the rank's
 *            shared-parameter gradient partials reduced to its subtree sum;
 *   exchange 1: rank j's subtree sum of rank r's owned parameter slice ->
 *            rank r (edpc_partials_pull, or NCCL send/recv inside phase 1);
 *   phase 1: G-leaf canonical tree + Adam on the owned slice only;
 *   exchange 2: the owned slices of the updated weights to every rank
 *            (edpc_weights_pull, or NCCL all-gather inside phase 1).
 * The trajectory is bit-identical to one context holding all 8 groups. */
int edpc_step_phase(edpc_ctx* ctx, int64_t i, int32_t phase, int32_t decompress);
int edpc_grad_partials(edpc_ctx* ctx, float** dev_ptr, int64_t* n_shared);
/* this context's lane groups [g_first, g_first + g_count) */
int edpc_ctx_groups(edpc_ctx* ctx, int32_t* g_first, int32_t* g_count);
/* this context's owned shared-parameter slice [off, off + len) */
int edpc_shard_range(edpc_ctx* ctx, int64_t* off, int64_t* len);
/* host copy of lane-group partials [g0, g0+ng) x n_shared (to_device 0: read) */
int edpc_partials_copy(edpc_ctx* ctx, int32_t g0, int32_t ng, float* host, int32_t to_device);
/* single-process multi-context exchanges (peer copies, stream-ordered):
 * dst <- src's subtree sum of dst's owned slice; dst <- src's owned weights */
int edpc_partials_pull(edpc_ctx* dst, edpc_ctx* src);
int edpc_weights_pull(edpc_ctx* dst, edpc_ctx* src);
/* hand produced columns [.., upto) to the encoder stream (phase-driven compress) */
int edpc_encode_pending(edpc_ctx* ctx, int64_t upto);
/* NCCL: rank 0 makes an id (128 bytes), every rank joins concurrently; after
 * that each model step runs both exchanges over NVLink inside the step (and
 * inside its CUDA graph) -- multi-process, one GPU per rank. */
int edpc_nccl_unique_id(uint8_t* out, int32_t cap);
int edpc_ctx_set_comm(edpc_ctx* ctx, const uint8_t* id, int32_t nranks, int32_t rank);

int edpc_sync(edpc_ctx* ctx);

/* Context buffers come from the device's stream-ordered memory pool and stay
 * cached there after edpc_ctx_destroy (the next context reuses them; no
 * reference counterpart -- the reference allocates host arrays per call).
 * Returns the cached, unused memory of `device` to the driver. */
int edpc_trim_pool(int32_t device);

/* test/debug read-back of internal fp32 buffers after a step:
 * 0 gradient partials [8][n_shared], 1 probs, 2 x_local, 3 x_lte, 4 x_global,
 * 5 local branch outputs [k][B][h_l], 6 global branch outputs, 7 d(embedded
 * context), 8 logits, 9 per-lane FDM Adam m [B][F'][F'], 10 shared Adam m,
 * 11 shared Adam v, 12 per-lane FDM U.  count must equal the buffer's
 * element count. */
int edpc_debug_read(edpc_ctx* ctx, int32_t which, float* out, int64_t count);
/* IFR analytics (ifr.py:59-104 ksg_mi): KSG neighbour
 * counts of already-jittered fp64 samples z [n][dz], y [n][dy] (dims <= 16,
 * 1 <= k <= 32) under the Chebyshev norm, on `device`: count_z/count_y [n]
 * (strict inequality against each sample's k-th joint distance, self
 * excluded) and the number of samples whose k-th distance is 0. */
int edpc_ksg_counts(const double* z, int32_t dz, const double* y, int32_t dy, int64_t n,
                    int32_t k, int32_t device, int64_t* count_z, int64_t* count_y,
                    int64_t* degenerate);
/* debug: make the fused weight-gradient/Adam kernels also write the reduced
 * gradient into partial slot 0 (slots 1..7 zeroed) so edpc_debug_read(0)
 * keeps returning partials whose canonical tree is the gradient */
int edpc_debug_keep_grads(edpc_ctx* ctx, int32_t keep);
/* the shared-parameter Adam kernel on host arrays: `steps` updates of w0 by
 * grads[t][n] (_kernels.py:18-32 adam_update; tests pin it to the reference) */
int edpc_debug_adam(const float* w0, const float* grads, int64_t n, int32_t steps, double lr,
                    double beta1, double beta2, double eps, float* w_out, float* m_out,
                    float* v_out);
/* bare tcgen05 GEMM microbenchmark on device operands (avg ms per launch) */
int edpc_bench_gemm(int32_t M, int32_t N, int32_t K, int32_t a_mn, int32_t b_mn, int32_t nsplit,
                    int32_t iters, double* ms);
/* one GEMM through the tcgen05 path on host arrays (tests):
 * C[M][N] = A . B, A [M][K] (a_mn 0) or [K][M] (a_mn 1), B [N][K] (b_mn 0)
 * or [K][N] (b_mn 1) */
/* Tests: the fp16-operand tcgen05 GEMM (A, B as IEEE half bits; lbo/sbo
 * override the MN-major descriptor strides, 0 = default). */
int edpc_debug_gemm_h(int32_t M, int32_t N, int32_t K, int32_t a_mn, int32_t b_mn,
                      const uint16_t* A, const uint16_t* B, float* C, int32_t lbo, int32_t sbo);
int edpc_debug_gemm(int32_t M, int32_t N, int32_t K, int32_t a_mn, int32_t b_mn, const float* A,
                    const float* B, float* C, int32_t dbg);

/* ------------------------------------------------------------ measurement
 * CUDA-event timing of kernel regions on the stream each kernel runs on
 * (used by bench.py for the live roofline).  Regions: 0 GEMM, 1 FDM fwd,
 * 2 FDM bwd+Adam, 3 shared Adam, 4 softmax+quantize, 5 encoder, 6 decoder,
 * 7 bias/LN column sums, 8 elementwise/LN, 9 embedding grad.
 * edpc_prof_read(region = -1) returns the number of kernel launches since
 * the last edpc_prof() call (profiling on or off). */
int edpc_prof(edpc_ctx* ctx, int enable);
/* device timer on the context's stream: op 0 start, op 1 stop (joins the
 * encoder stream), op 2 wait + elapsed milliseconds into *ms */
int edpc_timer(edpc_ctx* ctx, int32_t op, double* ms);
int edpc_prof_read(edpc_ctx* ctx, int32_t region, double* ms, int64_t* count);

#ifdef __cplusplus
}
#endif
#endif /* EDPC_B200_H */
