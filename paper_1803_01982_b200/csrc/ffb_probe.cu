// Live FP64 tensor-core peak probe for bench.py's roofline denominator: a
// register-only DMMA loop (mma.sync m8n8k4 f64, 8 independent accumulator
// chains per warp) on every SM, timed with CUDA events on the caller's stream.
// MEASURED_PEAKS.json carries no FP64 entry, so the denominator is measured in
// the same run, at the same clocks, as the kernels it divides.
#include <cuda_runtime.h>

#include "../../include/ffb200.h"
#include "ffb_common.cuh"

namespace ffb {
namespace {

__global__ void __launch_bounds__(256) dmma_peak_kernel(double* out, int iters) {
  const double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma_884(c[i][0], c[i][1], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;   // keeps the loop alive
}

}  // namespace
}  // namespace ffb

extern "C" int ffb_fp64_peak_probe(void* stream, int iters, double* tflops) {
  if (!tflops || iters < 1) return FFB_ERR_ARGUMENT;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaStream_t st = (cudaStream_t)stream;
  double* out = nullptr;
  if (cudaMallocAsync(&out, sizeof(double), st) != cudaSuccess) return FFB_ERR_CUDA;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const dim3 grid(2 * sms), block(256);
  ffb::dmma_peak_kernel<<<grid, block, 0, st>>>(out, 64);   // warm-up
  cudaEventRecord(e0, st);
  ffb::dmma_peak_kernel<<<grid, block, 0, st>>>(out, iters);
  cudaEventRecord(e1, st);
  cudaError_t e = cudaEventSynchronize(e1);
  float ms = 0.f;
  if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFreeAsync(out, st);
  if (e != cudaSuccess || ms <= 0.f) return FFB_ERR_CUDA;
  // 8 DMMAs of 8 x 8 x 4 (2 flop per multiply-add) per warp per iteration
  const double flops = 2.0 * 256.0 * 8.0 * (double)iters * grid.x * (block.x / 32);
  *tflops = flops / (ms * 1e-3) / 1e12;
  return FFB_OK;
}
