// Microbenchmarks behind DESIGN's latency budgets (B200): dependent-chain
// latency and per-SM throughput of DFMA, DADD, SHFL(64-bit), LDS/STS, F2F, MUFU.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe_bin/dp_probe tools/probe/dp_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat_dfma(double* out, long long* cyc, double a, double b) {
  double x = a;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 64; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) x = fma(x, b, a);
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void lat_dadd(double* out, long long* cyc, double a, double b) {
  double x = a;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 64; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) x = x + b;
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void lat_shfl(double* out, long long* cyc, double a) {
  double x = a + threadIdx.x;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 64; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) x = __shfl_xor_sync(0xffffffffu, x, 1 + (j & 15));
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void lat_shfl_add(double* out, long long* cyc, double a) {
  double x = a + threadIdx.x;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 64; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) x += __shfl_xor_sync(0xffffffffu, x, 1 + (j & 15));
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void lat_f2f(double* out, long long* cyc, double a) {
  double x = a;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 64; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float f = (float)x;
      x = (double)f;
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void lat_rsqrtf(float* out, long long* cyc, float a) {
  float x = a;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 64; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) x = rsqrtf(x);
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void lat_lds(double* out, long long* cyc) {
  __shared__ int nxt[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) nxt[i] = (i + 32) & 1023;
  __syncthreads();
  int p = threadIdx.x;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 64; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) p = nxt[p];
  }
  long long t1 = clock64();
  out[threadIdx.x] = p;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

// throughput: W warps per CTA, each with 8 independent DFMA chains
__global__ void thr_dfma(double* out, long long* cyc, double a, double b) {
  double x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = a + j;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = fma(x[j], b, a);
  }
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += x[j];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

// smem throughput: every warp streams 64-bit loads+stores over its own region
__global__ void thr_smem(double* out, long long* cyc) {
  extern __shared__ double sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* base = sm + warp * 32 * 16;
  for (int q = 0; q < 16; ++q) base[lane + 32 * q] = lane + q;
  __syncthreads();
  long long t0 = clock64();
  double acc = 0;
#pragma unroll 1
  for (int i = 0; i < 64; ++i) {
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      double v = base[lane + 32 * q];
      base[lane + 32 * q] = v + 1.0;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  out[threadIdx.x] = acc + base[lane];
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 16);
  cudaMallocManaged(&cyc, 64);
  auto rep = [&](const char* name, double per) {
    cudaDeviceSynchronize();
    printf("%-28s %8.1f cycles per op\n", name, cyc[0] / per);
  };
  lat_dfma<<<1, 32>>>(out, cyc, 1.0, 0.999); rep("DFMA dependent latency", 1024.0);
  lat_dadd<<<1, 32>>>(out, cyc, 1.0, 0.999); rep("DADD dependent latency", 1024.0);
  lat_shfl<<<1, 32>>>(out, cyc, 1.0); rep("SHFL f64 (2x32) latency", 1024.0);
  lat_shfl_add<<<1, 32>>>(out, cyc, 1.0); rep("SHFL f64 + DADD latency", 1024.0);
  lat_f2f<<<1, 32>>>(out, cyc, 1.5); rep("F2F f64->f32->f64 pair", 512.0);
  lat_rsqrtf<<<1, 32>>>((float*)out, cyc, 1.5f); rep("MUFU.RSQ f32 latency", 1024.0);
  lat_lds<<<1, 32>>>(out, cyc); rep("LDS dependent latency", 1024.0);
  for (int w : {1, 2, 4, 8, 16, 32}) {
    thr_dfma<<<1, 32 * w>>>(out, cyc, 1.0, 0.999);
    cudaDeviceSynchronize();
    const double instr = 256.0 * 8 * w;
    printf("DFMA throughput %2d warps/SM: %6.2f cycles per warp-DFMA per SM  (%.1f DFMA lanes/clk/SM)\n", w,
           cyc[0] / instr, instr * 32 / cyc[0]);
  }
  for (int w : {1, 4, 8, 16}) {
    cudaFuncSetAttribute(thr_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    thr_smem<<<1, 32 * w, w * 32 * 16 * 8>>>(out, cyc);
    cudaDeviceSynchronize();
    const double bytes = 64.0 * 16 * 2 * 256 * w;
    printf("smem LDS+STS.64 %2d warps: %.1f bytes/clk/SM\n", w, bytes / cyc[0]);
  }
  return 0;
}
