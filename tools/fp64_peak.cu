// FP64 peak probes for the roofline denominator: DMMA (mma.sync m8n8k4 f64) and DFMA.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}
__global__ void dfma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-9;
  double c[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) c[i] = fma(c[i], b, a);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += c[i];
  if (s == 12345.678) out[0] = s;
}
int main() {
  int dev = 0, sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out; cudaMalloc(&out, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 20000;
  for (int warps : {4, 8, 16, 32}) {
    for (int bpsm : {1, 2}) {
      dim3 grid(sms * bpsm), block(32 * warps);
      dmma_loop<<<grid, block>>>(out, 100);
      cudaEventRecord(e0);
      dmma_loop<<<grid, block>>>(out, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 256 * 8 * (double)iters * grid.x * warps;
      printf("DMMA warps/cta=%d ctas/sm=%d : %.2f TFLOP/s\n", warps, bpsm, flops / ms / 1e9);
    }
  }
  for (int warps : {8, 16, 32}) {
    dim3 grid(sms * 2), block(32 * warps);
    dfma_loop<<<grid, block>>>(out, 100);
    cudaEventRecord(e0);
    dfma_loop<<<grid, block>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 16 * (double)iters * grid.x * block.x;
    printf("DFMA warps/cta=%d ctas/sm=2 : %.2f TFLOP/s\n", warps, flops / ms / 1e9);
  }
  printf("SMs=%d err=%s\n", sms, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
