// Kernel-to-kernel gap inside a CUDA graph on one stream, with and without
// programmatic dependent launch (the secondary waits with griddepcontrol.wait).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe_bin/pdl_probe tools/probe/pdl_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void tiny(double* x, int n, int spin) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  double v = i < n ? x[i] : 0.0;
  for (int k = 0; k < spin; ++k) v = fma(v, 1.0000001, 1e-9);
  if (i < n) x[i] = v;
}

static float run(bool pdl, int nk, int grid, int spin, double* x, int n) {
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
  for (int k = 0; k < nk; ++k) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, tiny, x, n, spin);
  }
  cudaStreamEndCapture(st, &g);
  cudaGraphInstantiate(&ge, g, 0);
  for (int w = 0; w < 3; ++w) cudaGraphLaunch(ge, st);
  cudaStreamSynchronize(st);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, st);
  for (int r = 0; r < 10; ++r) cudaGraphLaunch(ge, st);
  cudaEventRecord(e1, st);
  cudaStreamSynchronize(st);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("  %s: %d kernels, grid %d, spin %d: %.2f us per kernel (err %s)\n", pdl ? "PDL   " : "serial", nk, grid,
         spin, ms * 1e3 / (10.0 * nk), cudaGetErrorString(cudaGetLastError()));
  return ms;
}

int main() {
  double* x;
  const int n = 148 * 256;
  cudaMalloc(&x, n * sizeof(double));
  cudaMemset(x, 0, n * sizeof(double));
  for (int grid : {1, 148}) {
    for (int spin : {0, 2000}) {
      run(false, 200, grid, spin, x, n);
      run(true, 200, grid, spin, x, n);
    }
  }
  return 0;
}
