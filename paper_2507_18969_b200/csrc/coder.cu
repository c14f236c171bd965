// Coder parity entry points: the device quantizer / encoder / decoder exposed
// one call at a time with caller-owned registers, mirroring quantize_rows,
// ArithmeticEncoder.encode_rows/finish and ArithmeticDecoder.__init__/
// decode_rows (pkg/src/edpc/coder.py:83-353).  The product path uses the very
// same device functions (coder.cuh) from the step kernels in model.cu.
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <string>
#include <vector>

#include "coder.cuh"
#include "common.cuh"

namespace edpc {

namespace {
thread_local std::string g_last_error;
}

void set_error(const std::string& msg) { g_last_error = msg; }
const char* last_error() { return g_last_error.c_str(); }

struct DevBuf {
  void* p = nullptr;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  int alloc(size_t bytes) {
    if (bytes == 0) bytes = 16;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) {
      set_error(std::string("cudaMalloc: ") + cudaGetErrorString(e));
      p = nullptr;
      return EDPC_ERR_NOMEM;
    }
    return EDPC_OK;
  }
  template <typename T>
  T* as() {
    return reinterpret_cast<T*>(p);
  }
};

static int use_device(int device) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    set_error("no CUDA device available (the B200 path has no CPU fallback)");
    return EDPC_ERR_CUDA;
  }
  EDPC_CHECK_ARG(device >= 0 && device < n, "device ordinal out of range");
  EDPC_CUDA_TRY(cudaSetDevice(device));
  return EDPC_OK;
}

// ---------------------------------------------------------------- kernels

template <bool kF64>
__global__ void k_quantize_rows(const void* __restrict__ probs, int64_t n,
                                uint32_t* __restrict__ cums) {
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (row >= n) return;
  const int lane = threadIdx.x & 31;
  double p[8];
  if (kF64) {
    const double* src = reinterpret_cast<const double*>(probs) + row * 256 + lane * 8;
#pragma unroll
    for (int j = 0; j < 8; ++j) p[j] = src[j];
  } else {
    const float* src = reinterpret_cast<const float*>(probs) + row * 256 + lane * 8;
#pragma unroll
    for (int j = 0; j < 8; ++j) p[j] = (double)src[j];
  }
  int freq[8];
  warp_quantize<kF64>(p, freq);
  uint32_t cum[8];
  warp_cdf(freq, cum);
  uint32_t* dst = cums + row * 257;
#pragma unroll
  for (int j = 0; j < 8; ++j) dst[lane * 8 + j] = cum[j];
  if (lane == 31) dst[256] = cum[7] + (uint32_t)freq[7];
}

__global__ void k_encode_rows(int64_t* st_io, uint32_t* words, int64_t cap_words,
                              const uint32_t* __restrict__ cums, const int32_t* __restrict__ sym,
                              int64_t n) {
  EncState st{(uint64_t)st_io[0], (uint64_t)st_io[1], (uint64_t)st_io[2], (uint64_t)st_io[3]};
  BitWriter w;
  w.open(words, st.bitpos, (uint64_t)cap_words);
  for (int64_t r = 0; r < n; ++r) {
    int s = sym[r];
    enc_symbol(st, w, cums[r * 257 + s], cums[r * 257 + s + 1]);
  }
  w.close();
  st_io[0] = (int64_t)st.low;
  st_io[1] = (int64_t)st.high;
  st_io[2] = (int64_t)st.pending;
  st_io[3] = (int64_t)w.bitpos;
}

__global__ void k_encode_finish(int64_t* st_io, uint32_t* words, int64_t cap_words) {
  EncState st{(uint64_t)st_io[0], (uint64_t)st_io[1], (uint64_t)st_io[2], (uint64_t)st_io[3]};
  BitWriter w;
  w.open(words, st.bitpos, (uint64_t)cap_words);
  enc_finish(st, w);
  w.close();
  st_io[2] = 0;
  st_io[3] = (int64_t)w.bitpos;
}

__global__ void k_decoder_init(int64_t* st_io, const uint8_t* data, int64_t bit_length) {
  uint64_t code = 0;
  for (int i = 0; i < 32; ++i) code = (code << 1) | read_bit(data, bit_length, i);
  st_io[0] = 0;
  st_io[1] = (int64_t)kMask32;
  st_io[2] = (int64_t)code;
  st_io[3] = 32;
}

// one warp; rows decoded serially, each symbol search warp-parallel
__global__ void k_decode_rows(int64_t* st_io, const uint8_t* __restrict__ data,
                              int64_t bit_length, const uint32_t* __restrict__ cums, int64_t n,
                              int32_t* out, int64_t* done) {
  const int lane = threadIdx.x & 31;
  DecState st{(uint64_t)st_io[0], (uint64_t)st_io[1], (uint64_t)st_io[2], st_io[3]};
  int64_t r = 0;
  bool ok = true;
  for (; r < n; ++r) {
    uint32_t cum[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) cum[j] = cums[r * 257 + lane * 8 + j];
    uint64_t span = st.high - st.low + 1;
    uint64_t value = dec_value(st, span);
    uint32_t c_lo, c_hi;
    int s = warp_find_symbol(cum, value, c_lo, c_hi);
    ok = dec_advance(st, data, bit_length, span, c_lo, c_hi);
    if (!ok) {
      if (lane == 0) out[r] = -1;
      break;
    }
    if (lane == 0) out[r] = s;
  }
  if (lane == 0) {
    st_io[0] = (int64_t)st.low;
    st_io[1] = (int64_t)st.high;
    st_io[2] = (int64_t)st.code;
    st_io[3] = st.bitpos;
    *done = r;
  }
}

}  // namespace edpc

using namespace edpc;

extern "C" {

const char* edpc_last_error(void) { return last_error(); }
int edpc_abi_version(void) { return EDPC_ABI_VERSION; }

int edpc_device_count(int* count) {
  EDPC_CHECK_ARG(count, "null count");
  cudaError_t e = cudaGetDeviceCount(count);
  if (e != cudaSuccess) {
    *count = 0;
    set_error(std::string("cudaGetDeviceCount: ") + cudaGetErrorString(e));
    return EDPC_ERR_CUDA;
  }
  return EDPC_OK;
}

int edpc_quantize_rows(int device, const void* probs, int64_t n, int dtype, uint32_t* cums) {
  EDPC_CHECK_ARG(n >= 0 && (dtype == 0 || dtype == 1), "bad quantize arguments");
  EDPC_CHECK_ARG(n == 0 || (probs && cums), "null buffer");
  if (n == 0) return EDPC_OK;
  EDPC_TRY(use_device(device));
  size_t in_bytes = (size_t)n * 256 * (dtype ? 8 : 4);
  DevBuf din, dout;
  EDPC_TRY(din.alloc(in_bytes));
  EDPC_TRY(dout.alloc((size_t)n * 257 * 4));
  EDPC_CUDA_TRY(cudaMemcpy(din.p, probs, in_bytes, cudaMemcpyHostToDevice));
  const int rows_per_block = 8;
  dim3 grid((unsigned)cdiv(n, rows_per_block));
  if (dtype)
    k_quantize_rows<true><<<grid, rows_per_block * 32>>>(din.p, n, dout.as<uint32_t>());
  else
    k_quantize_rows<false><<<grid, rows_per_block * 32>>>(din.p, n, dout.as<uint32_t>());
  EDPC_CUDA_TRY(cudaGetLastError());
  EDPC_CUDA_TRY(cudaMemcpy(cums, dout.p, (size_t)n * 257 * 4, cudaMemcpyDeviceToHost));
  return EDPC_OK;
}

static int round_words(int64_t cap) { return (int)((cap + 3) / 4); }

int edpc_encode_rows(int device, int64_t* enc_state, uint8_t* buf, int64_t cap,
                     const uint32_t* cums, const int32_t* symbols, int64_t n) {
  EDPC_CHECK_ARG(enc_state && buf && cap > 0 && n >= 0, "bad encode arguments");
  EDPC_CHECK_ARG(n == 0 || (cums && symbols), "null buffer");
  int64_t need_bits = enc_state[3] + 18 * n + enc_state[2] + 64;
  EDPC_CHECK_ARG(need_bits <= cap * 8, "encoder buffer too small");
  if (n == 0) return EDPC_OK;
  EDPC_TRY(use_device(device));
  DevBuf dst, dbuf, dc, ds;
  int64_t wbytes = (int64_t)round_words(cap) * 4;
  EDPC_TRY(dst.alloc(32));
  EDPC_TRY(dbuf.alloc(wbytes));
  EDPC_TRY(dc.alloc((size_t)n * 257 * 4));
  EDPC_TRY(ds.alloc((size_t)n * 4));
  EDPC_CUDA_TRY(cudaMemset(dbuf.p, 0, wbytes));
  EDPC_CUDA_TRY(cudaMemcpy(dbuf.p, buf, cap, cudaMemcpyHostToDevice));
  EDPC_CUDA_TRY(cudaMemcpy(dst.p, enc_state, 32, cudaMemcpyHostToDevice));
  EDPC_CUDA_TRY(cudaMemcpy(dc.p, cums, (size_t)n * 257 * 4, cudaMemcpyHostToDevice));
  EDPC_CUDA_TRY(cudaMemcpy(ds.p, symbols, (size_t)n * 4, cudaMemcpyHostToDevice));
  k_encode_rows<<<1, 1>>>(dst.as<int64_t>(), dbuf.as<uint32_t>(), wbytes / 4, dc.as<uint32_t>(),
                          ds.as<int32_t>(), n);
  EDPC_CUDA_TRY(cudaGetLastError());
  EDPC_CUDA_TRY(cudaMemcpy(enc_state, dst.p, 32, cudaMemcpyDeviceToHost));
  EDPC_CUDA_TRY(cudaMemcpy(buf, dbuf.p, cap, cudaMemcpyDeviceToHost));
  return EDPC_OK;
}

int edpc_encode_finish(int device, int64_t* enc_state, uint8_t* buf, int64_t cap,
                       int64_t* bit_length) {
  EDPC_CHECK_ARG(enc_state && buf && bit_length, "bad finish arguments");
  EDPC_CHECK_ARG(enc_state[3] + enc_state[2] + 8 <= cap * 8, "encoder buffer too small");
  EDPC_TRY(use_device(device));
  DevBuf dst, dbuf;
  int64_t wbytes = (int64_t)round_words(cap) * 4;
  EDPC_TRY(dst.alloc(32));
  EDPC_TRY(dbuf.alloc(wbytes));
  EDPC_CUDA_TRY(cudaMemset(dbuf.p, 0, wbytes));
  EDPC_CUDA_TRY(cudaMemcpy(dbuf.p, buf, cap, cudaMemcpyHostToDevice));
  EDPC_CUDA_TRY(cudaMemcpy(dst.p, enc_state, 32, cudaMemcpyHostToDevice));
  k_encode_finish<<<1, 1>>>(dst.as<int64_t>(), dbuf.as<uint32_t>(), wbytes / 4);
  EDPC_CUDA_TRY(cudaGetLastError());
  EDPC_CUDA_TRY(cudaMemcpy(enc_state, dst.p, 32, cudaMemcpyDeviceToHost));
  EDPC_CUDA_TRY(cudaMemcpy(buf, dbuf.p, cap, cudaMemcpyDeviceToHost));
  *bit_length = enc_state[3];
  return EDPC_OK;
}

int edpc_decoder_init(int device, int64_t* dec_state, const uint8_t* data, int64_t nbytes,
                      int64_t bit_length) {
  EDPC_CHECK_ARG(dec_state && nbytes >= 0 && bit_length >= 0, "bad decoder arguments");
  if (bit_length > nbytes * 8) {
    set_error("bit length exceeds payload");
    return EDPC_ERR_CODER;
  }
  EDPC_TRY(use_device(device));
  DevBuf dst, dd;
  EDPC_TRY(dst.alloc(32));
  EDPC_TRY(dd.alloc(nbytes + 16));
  EDPC_CUDA_TRY(cudaMemset(dd.p, 0, nbytes + 16));
  if (nbytes) EDPC_CUDA_TRY(cudaMemcpy(dd.p, data, nbytes, cudaMemcpyHostToDevice));
  k_decoder_init<<<1, 1>>>(dst.as<int64_t>(), dd.as<uint8_t>(), bit_length);
  EDPC_CUDA_TRY(cudaGetLastError());
  EDPC_CUDA_TRY(cudaMemcpy(dec_state, dst.p, 32, cudaMemcpyDeviceToHost));
  return EDPC_OK;
}

int edpc_decode_rows(int device, int64_t* dec_state, const uint8_t* data, int64_t nbytes,
                     int64_t bit_length, const uint32_t* cums, int64_t n, int32_t* out,
                     int64_t* done) {
  EDPC_CHECK_ARG(dec_state && done && n >= 0 && nbytes >= 0, "bad decode arguments");
  EDPC_CHECK_ARG(n == 0 || (cums && out), "null buffer");
  *done = 0;
  if (n == 0) return EDPC_OK;
  EDPC_TRY(use_device(device));
  DevBuf dst, dd, dc, dout, ddone;
  EDPC_TRY(dst.alloc(32));
  EDPC_TRY(dd.alloc(nbytes + 16));
  EDPC_TRY(dc.alloc((size_t)n * 257 * 4));
  EDPC_TRY(dout.alloc((size_t)n * 4));
  EDPC_TRY(ddone.alloc(8));
  EDPC_CUDA_TRY(cudaMemset(dd.p, 0, nbytes + 16));
  if (nbytes) EDPC_CUDA_TRY(cudaMemcpy(dd.p, data, nbytes, cudaMemcpyHostToDevice));
  EDPC_CUDA_TRY(cudaMemcpy(dst.p, dec_state, 32, cudaMemcpyHostToDevice));
  EDPC_CUDA_TRY(cudaMemcpy(dc.p, cums, (size_t)n * 257 * 4, cudaMemcpyHostToDevice));
  k_decode_rows<<<1, 32>>>(dst.as<int64_t>(), dd.as<uint8_t>(), bit_length, dc.as<uint32_t>(), n,
                           dout.as<int32_t>(), ddone.as<int64_t>());
  EDPC_CUDA_TRY(cudaGetLastError());
  EDPC_CUDA_TRY(cudaMemcpy(dec_state, dst.p, 32, cudaMemcpyDeviceToHost));
  EDPC_CUDA_TRY(cudaMemcpy(done, ddone.p, 8, cudaMemcpyDeviceToHost));
  EDPC_CUDA_TRY(cudaMemcpy(out, dout.p, (size_t)n * 4, cudaMemcpyDeviceToHost));
  if (*done != n) {
    set_error("bitstream exhausted at symbol " + std::to_string(*done) + " of this batch");
    return EDPC_ERR_CODER;
  }
  return EDPC_OK;
}

}  // extern "C"
