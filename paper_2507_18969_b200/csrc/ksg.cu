// KSG k-nearest-neighbour mutual-information counts on the GPU (SURVEY.md
// §8f rank 4; the reference's IFR analytics, `ifr.py:59-104`).
//
// For every sample i of the (already jittered) sample matrices z [n][dz],
// y [n][dy], under the Chebyshev norm:
//   eps_i     = k-th smallest of max(|z_i - z_j|_inf, |y_i - y_j|_inf), j != i
//   count_z_i = #{j != i : |z_i - z_j|_inf < eps_i}, count_y_i likewise
// (ifr.py:85-95: strict inequality; the self distance 0 is counted iff
// eps_i > 0 and then subtracted, which equals excluding j = i).  Everything
// is fp64 with the same operations as numpy (subtract, abs, max), so the
// counts are exactly the reference's; the digamma sum stays on the host.
//
// O(n^2 (dz + dy)) work: a CTA of 8 warps takes 8 queries (one per warp) and
// streams the n samples through shared memory in tiles of 128; each lane
// keeps a sorted register list of its k smallest joint distances, the warp
// then extracts the k-th smallest of the 32 lists by k rounds of a warp
// argmin.  A second sweep counts.  HBM traffic is n (dz + dy) 8 B per CTA
// (L2-resident for n <= 1e5); the bound is the fp64 compare/max rate.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <string>

#include "common.cuh"

namespace edpc {

constexpr int kKsgMaxD = 16;       // dz, dy <= 16 (the IFR study uses 8)
constexpr int kKsgMaxK = 32;       // neighbours
constexpr int kKsgWarps = 8;       // queries per CTA
constexpr int kKsgTile = 128;      // samples per shared-memory tile (2 x 16 KB)

__device__ __forceinline__ double cheb(const double* a, const double* b, int d) {
  double m = 0.0;
  for (int c = 0; c < d; ++c) m = fmax(m, fabs(a[c] - b[c]));
  return m;
}

__global__ void __launch_bounds__(32 * kKsgWarps)
k_ksg_counts(const double* __restrict__ z, int dz, const double* __restrict__ y, int dy, int64_t n,
             int k, int64_t* __restrict__ cz, int64_t* __restrict__ cy,
             unsigned long long* __restrict__ degenerate) {
  __shared__ double tz[kKsgTile * kKsgMaxD];
  __shared__ double ty[kKsgTile * kKsgMaxD];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * kKsgWarps + warp;
  const bool live = i < n;
  double qz[kKsgMaxD], qy[kKsgMaxD];
  for (int c = 0; c < dz; ++c) qz[c] = live ? z[i * dz + c] : 0.0;
  for (int c = 0; c < dy; ++c) qy[c] = live ? y[i * dy + c] : 0.0;
  // per-lane sorted list of the k smallest joint distances seen
  double best[kKsgMaxK];
  for (int q = 0; q < kKsgMaxK; ++q) best[q] = INFINITY;
  for (int64_t t0 = 0; t0 < n; t0 += kKsgTile) {
    const int cnt = (int)(n - t0 < kKsgTile ? n - t0 : kKsgTile);
    __syncthreads();
    for (int e = threadIdx.x; e < cnt * dz; e += blockDim.x) tz[e] = z[t0 * dz + e];
    for (int e = threadIdx.x; e < cnt * dy; e += blockDim.x) ty[e] = y[t0 * dy + e];
    __syncthreads();
    if (!live) continue;
    for (int jj = lane; jj < cnt; jj += 32) {
      if (t0 + jj == i) continue;  // self excluded from the joint ranking (ifr.py:90)
      const double dj = fmax(cheb(qz, tz + jj * dz, dz), cheb(qy, ty + jj * dy, dy));
      if (dj < best[k - 1]) {  // insertion into the sorted list
        int p = k - 1;
        while (p > 0 && best[p - 1] > dj) {
          best[p] = best[p - 1];
          --p;
        }
        best[p] = dj;
      }
    }
  }
  // k-th smallest over the warp: k rounds of argmin over the lanes' heads
  double eps = INFINITY;
  int head = 0;
  for (int r = 0; r < k; ++r) {
    double v = head < k ? best[head] : INFINITY;
    int who = lane;
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, v, o);
      const int ow = __shfl_xor_sync(0xffffffffu, who, o);
      if (ov < v || (ov == v && ow < who)) {
        v = ov;
        who = ow;
      }
    }
    eps = v;
    if (lane == who) ++head;
  }
  // counts with strict inequality against eps
  int64_t nz = 0, ny = 0;
  for (int64_t t0 = 0; t0 < n; t0 += kKsgTile) {
    const int cnt = (int)(n - t0 < kKsgTile ? n - t0 : kKsgTile);
    __syncthreads();
    for (int e = threadIdx.x; e < cnt * dz; e += blockDim.x) tz[e] = z[t0 * dz + e];
    for (int e = threadIdx.x; e < cnt * dy; e += blockDim.x) ty[e] = y[t0 * dy + e];
    __syncthreads();
    if (!live) continue;
    for (int jj = lane; jj < cnt; jj += 32) {
      if (t0 + jj == i) continue;
      nz += cheb(qz, tz + jj * dz, dz) < eps;
      ny += cheb(qy, ty + jj * dy, dy) < eps;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    nz += __shfl_xor_sync(0xffffffffu, nz, o);
    ny += __shfl_xor_sync(0xffffffffu, ny, o);
  }
  if (live && lane == 0) {
    cz[i] = nz;
    cy[i] = ny;
    if (eps == 0.0) atomicAdd(degenerate, 1ull);  // integer: order-independent
  }
}

}  // namespace edpc

using namespace edpc;

extern "C" int edpc_ksg_counts(const double* z, int32_t dz, const double* y, int32_t dy, int64_t n,
                               int32_t k, int32_t device, int64_t* count_z, int64_t* count_y,
                               int64_t* degenerate) {
  EDPC_CHECK_ARG(z && y && count_z && count_y && degenerate, "null argument");
  EDPC_CHECK_ARG(dz >= 1 && dz <= kKsgMaxD && dy >= 1 && dy <= kKsgMaxD,
                 "sample dims must be in [1, 16]");
  EDPC_CHECK_ARG(k >= 1 && k <= kKsgMaxK, "neighbours must be in [1, 32]");
  EDPC_CHECK_ARG(n >= k + 1, "not enough samples for the requested neighbour count");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    set_error("no CUDA device available (the B200 path has no CPU fallback)");
    return EDPC_ERR_CUDA;
  }
  EDPC_CHECK_ARG(device >= 0 && device < ndev, "device ordinal out of range");
  EDPC_CUDA_TRY(cudaSetDevice(device));
  double *dz_, *dy_;
  int64_t *cz, *cy;
  unsigned long long* dg;
  EDPC_CUDA_TRY(cudaMalloc(&dz_, (size_t)n * dz * 8));
  EDPC_CUDA_TRY(cudaMalloc(&dy_, (size_t)n * dy * 8));
  EDPC_CUDA_TRY(cudaMalloc(&cz, (size_t)n * 8));
  EDPC_CUDA_TRY(cudaMalloc(&cy, (size_t)n * 8));
  EDPC_CUDA_TRY(cudaMalloc(&dg, 8));
  cudaError_t e = cudaMemcpy(dz_, z, (size_t)n * dz * 8, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(dy_, y, (size_t)n * dy * 8, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemset(dg, 0, 8);
  if (e == cudaSuccess) {
    k_ksg_counts<<<(unsigned)cdiv(n, (int64_t)kKsgWarps), 32 * kKsgWarps>>>(dz_, dz, dy_, dy, n, k,
                                                                          cz, cy, dg);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpy(count_z, cz, (size_t)n * 8, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(count_y, cy, (size_t)n * 8, cudaMemcpyDeviceToHost);
  unsigned long long d = 0;
  if (e == cudaSuccess) e = cudaMemcpy(&d, dg, 8, cudaMemcpyDeviceToHost);
  cudaFree(dz_);
  cudaFree(dy_);
  cudaFree(cz);
  cudaFree(cy);
  cudaFree(dg);
  EDPC_CUDA_TRY(e);
  *degenerate = (int64_t)d;
  return EDPC_OK;
}
