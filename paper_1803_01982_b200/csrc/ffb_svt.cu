// SVT / IALM iteration kernels around the partial SVD (ffsrqr/nuclear.py:91-191).
//
// One IALM iteration outside the partial SVD is a handful of elementwise passes
// over m x n matrices in the reference (soft-shrink, residual Z, multiplier
// update, the next SVD input, ||Z||_F).  Here they are ONE HBM-bound pass:
// read M, X, Y (+ mask), write E, Y, W = M - E + Y / mu_next, and a
// deterministic per-CTA partial of ||Z||^2 (fixed grid, fixed-order tree, then
// a fixed-order sum of the partials), so results are bitwise reproducible.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/ffb200.h"
#include "ffb_common.cuh"

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ double block_sum_fixed(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
  return s;
}

// mode 0: RPCA, E = sign(a) max(|a| - thresh, 0)   (nuclear.py:131)
// mode 1: matrix completion, E = mask ? 0 : a        (nuclear.py:174)
// with a = (M - X) + Y / mu;  Z = (M - X) - E;  Y += mu Z;  W = (M - E) + Y / mu_next
__global__ void __launch_bounds__(kThreads) ialm_update_kernel(
    int mode, const double* __restrict__ M, const double* __restrict__ X, double* __restrict__ Y,
    double* __restrict__ E, const uint8_t* __restrict__ mask, int64_t count, double mu,
    double thresh, double mu_next, double* __restrict__ W, double* __restrict__ partials) {
  __shared__ double red[kThreads / 32];
  double acc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += stride) {
    const double m = M[i], x = X[i], y = Y[i];
    const double mx = m - x;
    const double a = mx + y / mu;
    double e;
    if (mode == 0) {
      const double t = fabs(a) - thresh;
      e = t > 0.0 ? copysign(t, a) : 0.0;
      if (a == 0.0) e = 0.0;
    } else {
      e = mask[i] ? 0.0 : a;
    }
    const double z = mx - e;
    const double yn = y + mu * z;
    E[i] = e;
    Y[i] = yn;
    W[i] = (m - e) + yn / mu_next;
    acc = fma(z, z, acc);
  }
  const double s = block_sum_fixed(acc, red);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

__global__ void sum_partials_kernel(const double* __restrict__ partials, int np, double* out) {
  __shared__ double red[kThreads / 32];
  double acc = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) acc += partials[i];
  const double s = block_sum_fixed(acc, red);
  if (threadIdx.x == 0) out[0] = s;
}

__global__ void __launch_bounds__(kThreads) sumsq_kernel(const double* __restrict__ x,
                                                         int64_t count, double* partials) {
  __shared__ double red[kThreads / 32];
  double acc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += stride)
    acc = fma(x[i], x[i], acc);
  const double s = block_sum_fixed(acc, red);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

// out[:, j] = U[:, j] * (s[j] - shift), j < keep   (nuclear.py:96)
__global__ void shrink_cols_kernel(const double* __restrict__ U, int64_t ldu, int64_t m,
                                   int64_t keep, const double* __restrict__ s, double shift,
                                   double* __restrict__ out, int64_t ldo) {
  const int64_t total = m * keep;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = idx / m, i = idx - j * m;
    out[i + j * ldo] = U[i + j * ldu] * (s[j] - shift);
  }
}

int grid_for(int64_t count) {
  int g = (int)((count + kThreads - 1) / kThreads);
  return g < 1 ? 1 : (g > 4 * 148 ? 4 * 148 : g);
}

}  // namespace

extern "C" {

int ffb_svt_partials(void) { return 4 * 148; }

int ffb_ialm_update(void* stream, int mode, const double* M, const double* X, double* Y, double* E,
                    const uint8_t* mask, int64_t count, double mu, double thresh, double mu_next,
                    double* W, double* partials, double* zsq) {
  if (!M || !X || !Y || !E || !W || !partials || !zsq || (mode == 1 && !mask) || count < 0)
    return FFB_ERR_ARGUMENT;
  cudaStream_t st = (cudaStream_t)stream;
  const int g = grid_for(count);
  ialm_update_kernel<<<g, kThreads, 0, st>>>(mode, M, X, Y, E, mask, count, mu, thresh, mu_next, W,
                                             partials);
  sum_partials_kernel<<<1, kThreads, 0, st>>>(partials, g, zsq);
  return cudaGetLastError() == cudaSuccess ? FFB_OK : FFB_ERR_CUDA;
}

int ffb_sumsq(void* stream, const double* x, int64_t count, double* partials, double* out) {
  if (!x || !partials || !out || count < 0) return FFB_ERR_ARGUMENT;
  cudaStream_t st = (cudaStream_t)stream;
  const int g = grid_for(count);
  sumsq_kernel<<<g, kThreads, 0, st>>>(x, count, partials);
  sum_partials_kernel<<<1, kThreads, 0, st>>>(partials, g, out);
  return cudaGetLastError() == cudaSuccess ? FFB_OK : FFB_ERR_CUDA;
}

int ffb_shrink_cols(void* stream, const double* U, int64_t ldu, int64_t m, int64_t keep,
                    const double* s, double shift, double* out, int64_t ldo) {
  if (!U || !s || !out || m < 0 || keep < 0 || ldu < m || ldo < m) return FFB_ERR_ARGUMENT;
  if (m * keep == 0) return FFB_OK;
  shrink_cols_kernel<<<grid_for(m * keep), kThreads, 0, (cudaStream_t)stream>>>(U, ldu, m, keep, s,
                                                                                  shift, out, ldo);
  return cudaGetLastError() == cudaSuccess ? FFB_OK : FFB_ERR_CUDA;
}

}  // extern "C"
