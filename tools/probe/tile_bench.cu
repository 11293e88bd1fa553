// Microbenchmark of the 64x64 dense tile routines (ffb_tile64.cuh) on one CTA:
// cycles per call for the barrier-per-step versions vs the blocked ones.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1803_01982_b200/csrc tools/probe/tile_bench.cu -o tools/probe_bin/tile_bench
#include <cstdio>
#include <cstdlib>
#include <cmath>

#include "ffb_tile64.cuh"
using namespace ffb::tile64;

__global__ void __launch_bounds__(256, 1) bench(const double* G, const double* Q, int w, long long* cyc,
                                               double* out) {
  extern __shared__ double sm[];
  double* Rs = sm;
  double* Xs = Rs + 64 * kTL;
  double* A3 = Xs + 64 * kTL;
  double* A4 = A3 + 64 * kTL;
  double* S = A4 + 64 * kTL;
  double* buf = S + 1024;
  __shared__ double Dd[64];
  const int tid = threadIdx.x;
  Tile g;
  long long t0, t1;
  // old: chol_upper1 + inv_upper_blk
  for (int rep = 0; rep < 3; ++rep) {
    for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) {
      const int r = bi_of(tid) + i, c = bj_of(tid) + j;
      g.v[i][j] = (r < w && c < w) ? G[r * 64 + c] : 0.0;
    }
    __syncthreads();
    t0 = clock64();
    chol_upper1(g, w, Rs, buf);
    inv_upper_blk(Rs, w, Xs, S);
    __syncthreads();
    t1 = clock64();
    if (tid == 0) cyc[0] = t1 - t0;
  }
  for (int t = tid; t < 4096; t += 256) { out[t] = Rs[(t >> 6) * kTL + (t & 63)]; out[4096 + t] = Xs[(t >> 6) * kTL + (t & 63)]; }
  for (int rep = 0; rep < 3; ++rep) {
    for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) {
      const int r = bi_of(tid) + i, c = bj_of(tid) + j;
      g.v[i][j] = (r < w && c < w) ? G[r * 64 + c] : 0.0;
    }
    __syncthreads();
    t0 = clock64();
    chol_inv_blk(g, w, Rs, Xs, S);
    __syncthreads();
    t1 = clock64();
    if (tid == 0) cyc[1] = t1 - t0;
  }
  for (int t = tid; t < 4096; t += 256) { out[8192 + t] = Rs[(t >> 6) * kTL + (t & 63)]; out[12288 + t] = Xs[(t >> 6) * kTL + (t & 63)]; }
  // warp chol alone
  for (int rep = 0; rep < 3; ++rep) {
    for (int t = tid; t < 4096; t += 256) Rs[(t >> 6) * kTL + (t & 63)] = G[t];
    __syncthreads();
    t0 = clock64();
    if (tid < 32) warp_chol_inv16(Rs, Xs, 0, 16);
    __syncthreads();
    t1 = clock64();
    if (tid == 0) cyc[2] = t1 - t0;
  }
  // sign LU old / new
  for (int rep = 0; rep < 3; ++rep) {
    for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) {
      const int r = bi_of(tid) + i, c = bj_of(tid) + j;
      g.v[i][j] = (r < w && c < w) ? Q[r * 64 + c] : 0.0;
    }
    __syncthreads();
    t0 = clock64();
    sign_lu(g, w, Rs, Xs, Dd, buf);
    inv_upper_blk(Xs, w, A3, S);
    inv_unit_lower_blk(Rs, w, A4, S);
    __syncthreads();
    t1 = clock64();
    if (tid == 0) cyc[3] = t1 - t0;
  }
  for (int t = tid; t < 4096; t += 256) {
    out[16384 + t] = Rs[(t >> 6) * kTL + (t & 63)]; out[20480 + t] = Xs[(t >> 6) * kTL + (t & 63)];
    out[24576 + t] = A3[(t >> 6) * kTL + (t & 63)]; out[28672 + t] = A4[(t >> 6) * kTL + (t & 63)];
  }
}

int main(int argc, char** argv) {
  const int w = argc > 1 ? atoi(argv[1]) : 64;
  double *G, *Q, *out;
  long long* cyc;
  cudaMallocManaged(&G, 4096 * 8);
  cudaMallocManaged(&Q, 4096 * 8);
  cudaMallocManaged(&out, 49152 * 8);
  cudaMallocManaged(&cyc, 8 * 8);
  srand(1);
  double M[64 * 64];
  for (int i = 0; i < 4096; ++i) M[i] = (rand() / (double)RAND_MAX - 0.5);
  for (int i = 0; i < 64; ++i)
    for (int j = 0; j < 64; ++j) {
      double s = 0;
      for (int k = 0; k < 64; ++k) s += M[k * 64 + i] * M[k * 64 + j];
      G[i * 64 + j] = s + (i == j ? 64.0 : 0.0);
      Q[i * 64 + j] = 0.3 * M[i * 64 + j] + (i == j ? 0.5 : 0.0);
    }
  const size_t smem = sizeof(double) * (4 * 64 * kTL + 1024 + 256);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  bench<<<1, 256, smem>>>(G, Q, w, cyc, out);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  auto maxdiff = [&](int a, int b) {
    double m = 0, s = 0;
    for (int i = 0; i < 4096; ++i) { m = fmax(m, fabs(out[a + i] - out[b + i])); s = fmax(s, fabs(out[a + i])); }
    return m / (s > 0 ? s : 1);
  };
  printf("w=%d cycles: chol+inv old %lld blocked %lld (warp 16x16 %lld) | signlu+inv %lld\n", w,
         cyc[0], cyc[1], cyc[2], cyc[3]);
  printf("rel diff blocked vs old: R %.2e X %.2e\n", maxdiff(0, 8192), maxdiff(4096, 12288));
  return 0;
}
