// Small dense SVD (K14): one-sided block Jacobi (Hestenes) on the l x l
// triangular factor of tmp = A P Qhat_1 — replaces LAPACK dgesdd
// (ffsrqr/svd.py:79).  One-sided Jacobi on a triangular factor gives singular
// values to high RELATIVE accuracy, which the 1e-10 parity bound needs for the
// small end of the spectrum (a Gram-matrix eigensolver would lose u*kappa^2).
//
// Cooperative persistent kernel: the columns are split into nb (even) blocks of
// <= bs columns; each outer round, CTA p takes one block pair of a round-robin
// tournament, stages its 2*bs columns of M and of the accumulated V in shared
// memory, runs one inner cyclic sweep (2bs-1 parallel rounds, one warp per
// column pair) and writes them back; a grid barrier separates rounds.  Sweeps
// stop when the largest |x^T y| / (||x|| ||y||) seen in a sweep is <= tol.
#include <math.h>

#include "ffb_common.cuh"
#include "ffb_jacobi.cuh"

namespace ffb {

FFB_DEV uint32_t ld_acq(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
FFB_DEV void st_rel(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

// Sense/generation grid barrier; bar[0] = arrivals, bar[1] = generation.
FFB_DEV void grid_barrier(uint32_t* bar, uint32_t nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t gen = ld_acq(bar + 1);
    __threadfence();
    const uint32_t arrived = atomicAdd(bar, 1u) + 1u;
    if (arrived == nblocks) {
      atomicExch(bar, 0u);
      __threadfence();
      st_rel(bar + 1, gen + 1u);
    } else {
      while (ld_acq(bar + 1) == gen) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

// round-robin (circle method) player at position `pos` in round r for nb players
FFB_DEV int rr_player(int pos, int r, int nb) {
  if (pos == 0) return 0;
  return ((pos - 1 + r) % (nb - 1)) + 1;
}

__global__ void __launch_bounds__(1024) jacobi_kernel(JacobiArgs a) {
  extern __shared__ __align__(16) double sm[];
  const int l = a.l, bs = a.bs, nb = a.nb;
  const int W = 2 * bs;                 // local column slots
  double* Ms = sm;                      // [W][l]
  double* Vs = sm + (size_t)W * l;      // [W][l]
  __shared__ int gcol[64];              // global column of each local slot (-1 = empty)
  __shared__ double s_off;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int P = gridDim.x;
  uint32_t* bar = a.bar;

  for (int sweep = 0; sweep < a.max_sweeps; ++sweep) {
    if (tid == 0) s_off = 0.0;
    for (int r = 0; r < nb - 1; ++r) {
      // block pair of this CTA
      const int pa = rr_player(blockIdx.x, r, nb), pb = rr_player(nb - 1 - blockIdx.x, r, nb);
      if (tid < W) {
        const int blk = tid < bs ? pa : pb;
        const int c = blk * bs + (tid < bs ? tid : tid - bs);
        gcol[tid] = (c < (blk + 1) * bs && c < l) ? c : -1;
      }
      __syncthreads();
      for (int idx = tid; idx < W * l; idx += blockDim.x) {
        const int j = idx / l, i = idx % l;
        const int c = gcol[j];
        Ms[idx] = c >= 0 ? a.M[i + (int64_t)c * a.ldm] : 0.0;
        Vs[idx] = c >= 0 ? a.V[i + (int64_t)c * a.ldv] : 0.0;
      }
      __syncthreads();
      double off = 0.0;
      // inner cyclic sweep over the W local columns: W-1 rounds of W/2 pairs
      for (int t = 0; t < W - 1; ++t) {
        for (int pr = warp; pr < bs; pr += nwarps) {
          const int x = rr_player(pr, t, W), y = rr_player(W - 1 - pr, t, W);
          if (gcol[x] < 0 || gcol[y] < 0) continue;
          double* mx = Ms + (size_t)x * l;
          double* my = Ms + (size_t)y * l;
          double aa = 0.0, bb = 0.0, cc = 0.0;
          for (int i = lane; i < l; i += 32) {
            const double u = mx[i], v = my[i];
            aa = fma(u, u, aa);
            bb = fma(v, v, bb);
            cc = fma(u, v, cc);
          }
          aa = warp_sum(aa);
          bb = warp_sum(bb);
          cc = warp_sum(cc);
          if (!(fabs(cc) > a.tol * sqrt(aa * bb))) continue;
          off = fmax(off, fabs(cc) / sqrt(aa * bb));
          const double zeta = (bb - aa) / (2.0 * cc);
          const double tt = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double cs = 1.0 / sqrt(1.0 + tt * tt), sn = cs * tt;
          double* vx = Vs + (size_t)x * l;
          double* vy = Vs + (size_t)y * l;
          for (int i = lane; i < l; i += 32) {
            const double u = mx[i], v = my[i];
            mx[i] = cs * u - sn * v;
            my[i] = sn * u + cs * v;
            const double p = vx[i], q = vy[i];
            vx[i] = cs * p - sn * q;
            vy[i] = sn * p + cs * q;
          }
        }
        __syncthreads();
      }
      // write back
      for (int idx = tid; idx < W * l; idx += blockDim.x) {
        const int j = idx / l, i = idx % l;
        const int c = gcol[j];
        if (c >= 0) {
          a.M[i + (int64_t)c * a.ldm] = Ms[idx];
          a.V[i + (int64_t)c * a.ldv] = Vs[idx];
        }
      }
      // CTA-wide max of off -> global per-sweep max
      off = warp_max(off);
      if (lane == 0 && off > 0.0) atomicMax(reinterpret_cast<unsigned long long*>(&s_off),
                                            (unsigned long long)__double_as_longlong(off));
      __syncthreads();
      if (tid == 0 && s_off > 0.0)
        atomicMax(reinterpret_cast<unsigned long long*>(a.offmax + sweep),
                  (unsigned long long)__double_as_longlong(s_off));
      grid_barrier(bar, P);
    }
    const double om = *((volatile double*)(a.offmax + sweep));
    if (tid == 0 && blockIdx.x == 0) *a.sweeps = sweep + 1;
    if (!(om > a.tol)) break;
  }
}

// sigma_j = ||M[:, j]||; rank sort (descending, ties by index); outputs sorted
// sigma, U = M_j / sigma_j (zero column when sigma_j == 0) and V columns.
__global__ void jacobi_finish_kernel(const double* M, int64_t ldm, const double* V, int64_t ldv,
                                     int l, double* sig, double* U, int64_t ldu, double* Vo,
                                     int64_t ldvo, int* order) {
  extern __shared__ double nrm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  for (int j = warp; j < l; j += nw) {
    double acc = 0.0;
    for (int i = lane; i < l; i += 32) acc = fma(M[i + (int64_t)j * ldm], M[i + (int64_t)j * ldm], acc);
    acc = warp_sum(acc);
    if (lane == 0) nrm[j] = sqrt(acc);
  }
  __syncthreads();
  for (int j = tid; j < l; j += blockDim.x) {
    int rank = 0;
    const double sj = nrm[j];
    for (int q = 0; q < l; ++q) rank += (nrm[q] > sj) || (nrm[q] == sj && q < j);
    order[rank] = j;
    sig[rank] = sj;
  }
  __syncthreads();
  for (int idx = tid; idx < l * l; idx += blockDim.x) {
    const int r = idx / l, i = idx % l;
    const int j = order[r];
    const double s = nrm[j];
    U[i + (int64_t)r * ldu] = s > 0.0 ? M[i + (int64_t)j * ldm] / s : 0.0;
    Vo[i + (int64_t)r * ldvo] = V[i + (int64_t)j * ldv];
  }
}

int jacobi_block_size(int l) {
  int bs = (int)((200 * 1024) / ((size_t)l * 2 * 2 * sizeof(double)));
  if (bs > 32) bs = 32;
  if (bs < 1) bs = 1;
  return bs;
}

cudaError_t launch_jacobi_svd(cudaStream_t st, int sms, double* M, int64_t ldm, double* V,
                              int64_t ldv, int l, double* sig, double* U, int64_t ldu, double* Vo,
                              int64_t ldvo, uint32_t* bar, double* offmax, int* sweeps, int* order,
                              int max_sweeps) {
  const int bs = jacobi_block_size(l);
  int nb = (l + bs - 1) / bs;
  if (nb % 2) ++nb;
  if (nb < 2) nb = 2;
  const int P = nb / 2;
  (void)sms;
  JacobiArgs a{M, ldm, V, ldv, l, bs, nb, 1e-15 * sqrt((double)l), max_sweeps, bar, offmax, sweeps};
  const size_t smem = (size_t)2 * (2 * bs) * l * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(jacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
    attr = true;
  }
  cudaError_t e = cudaMemsetAsync(bar, 0, 2 * sizeof(uint32_t), st);
  if (e == cudaSuccess) e = cudaMemsetAsync(offmax, 0, sizeof(double) * max_sweeps, st);
  if (e != cudaSuccess) return e;
  const int threads = 32 * (bs < 4 ? 4 : bs);
  void* args[] = {&a};
  e = cudaLaunchCooperativeKernel((void*)jacobi_kernel, dim3(P), dim3(threads), args, smem, st);
  if (e != cudaSuccess) return e;
  jacobi_finish_kernel<<<1, 1024, sizeof(double) * (size_t)l, st>>>(M, ldm, V, ldv, l, sig, U, ldu,
                                                                    Vo, ldvo, order);
  return cudaGetLastError();
}

}  // namespace ffb
