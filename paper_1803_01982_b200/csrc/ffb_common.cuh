// Shared device helpers for the B200 Flip-Flop SRQR engine (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#define FFB_DEV __device__ __forceinline__

namespace ffb {

constexpr int kWarp = 32;

// Opt-in to more than 48 KB of dynamic shared memory for `kern` on the CURRENT
// device.  The attribute is per device, so a process driving several GPUs must
// set it once on each: `done` is the call site's bitmask of devices already set.
inline cudaError_t ensure_smem_optin(const void* kern, int bytes, std::atomic<unsigned long long>& done) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

// 1/x to ~1 ulp: MUFU reciprocal seed + two Newton steps (no IEEE division
// subroutine on the critical path of sequential factorizations)
FFB_DEV double fast_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  r = r * fma(-x, r, 2.0);
  r = r * fma(-x, r, 2.0);
  return r;
}

FFB_DEV double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

FFB_DEV double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Deterministic block-wide sum (fixed tree order). `red` needs blockDim/32 doubles.
FFB_DEV double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double t = 0.0;
  if (wid == 0) {
    t = lane < nw ? red[lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) red[0] = t;
  }
  __syncthreads();
  t = red[0];
  __syncthreads();
  return t;
}

// (value, index) argmax with ties broken to the LOWEST index (np.argmax convention,
// ffsrqr/_kernels_numba.py:32-37).
struct ArgMax {
  double v;
  int64_t i;
};

FFB_DEV ArgMax argmax_better(ArgMax a, ArgMax b) {
  // a "wins" if strictly larger, or equal with lower index. NaN never wins.
  if (b.v > a.v || (b.v == a.v && b.i < a.i) || (a.i < 0)) return b.i < 0 ? a : b;
  return a;
}

FFB_DEV ArgMax warp_argmax(ArgMax a) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ArgMax b;
    b.v = __shfl_xor_sync(0xffffffffu, a.v, o);
    b.i = __shfl_xor_sync(0xffffffffu, a.i, o);
    a = argmax_better(a, b);
  }
  return a;
}

// `red_v`/`red_i` need blockDim/32 entries.
FFB_DEV ArgMax block_argmax(ArgMax a, double* red_v, int64_t* red_i) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  a = warp_argmax(a);
  __syncthreads();
  if (lane == 0) {
    red_v[wid] = a.v;
    red_i[wid] = a.i;
  }
  __syncthreads();
  if (wid == 0) {
    ArgMax t{-1.0, -1};
    if (lane < nw) t = ArgMax{red_v[lane], red_i[lane]};
    t = warp_argmax(t);
    if (lane == 0) {
      red_v[0] = t.v;
      red_i[0] = t.i;
    }
  }
  __syncthreads();
  ArgMax r{red_v[0], red_i[0]};
  __syncthreads();
  return r;
}

// FP64 tensor core: D(8x8) += A(8x4) * B(4x8), row.col (DMMA.8x8x4 on sm_100a).
// Fragment ownership (lane t): a = A[t/4][t%4], b = B[t%4][t/4],
// c0 = C[t/4][2*(t%4)], c1 = C[t/4][2*(t%4)+1].
FFB_DEV void dmma_884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

FFB_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 8-byte async copy global->shared with zero fill when !pred.
FFB_DEV void cp_async8(void* smem, const double* gmem, bool pred) {
  const int bytes = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(smem)),
               "l"(gmem), "r"(bytes));
}

// 16-byte async copy (both addresses 16B aligned), zero fill when !pred.
FFB_DEV void cp_async16(void* smem, const double* gmem, bool pred) {
  const int bytes = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)),
               "l"(gmem), "r"(bytes));
}

FFB_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }

template <int N>
FFB_DEV void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

}  // namespace ffb
