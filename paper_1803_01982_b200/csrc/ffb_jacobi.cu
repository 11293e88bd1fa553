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

// One Hestenes rotation of local columns x, y (M and V), warp-cooperative.  The
// pair is loaded into registers in one burst (NPL elements per lane, fully
// unrolled), rotated there and stored back, so a round costs one shared-memory
// latency instead of a dependent chain.  nrm[] caches squared column norms.
template <int NPL>
FFB_DEV void jacobi_pair(double* Ms, double* Vs, double* nrm, int l, int x, int y, double tol,
                         int lane, double& off) {
  double* mx = Ms + (size_t)x * l;
  double* my = Ms + (size_t)y * l;
  double* vx = Vs + (size_t)x * l;
  double* vy = Vs + (size_t)y * l;
  double X[NPL], Yv[NPL];
#pragma unroll
  for (int q = 0; q < NPL; ++q) {
    const int i = lane + 32 * q;
    X[q] = i < l ? mx[i] : 0.0;
    Yv[q] = i < l ? my[i] : 0.0;
  }
  double c0 = 0.0, c1 = 0.0;
#pragma unroll
  for (int q = 0; q < NPL; q += 2) {
    c0 = fma(X[q], Yv[q], c0);
    if (q + 1 < NPL) c1 = fma(X[q + 1], Yv[q + 1], c1);
  }
  const double c = warp_sum(c0 + c1);
  const double a = nrm[x], b = nrm[y];
  const double ab = sqrt(a * b);
  if (!(fabs(c) > tol * ab)) return;
  off = fmax(off, fabs(c) / ab);
  // rotation angle: only cs^2 + sn^2 = 1 must be exact; t itself may be approximate
  // (it only sets how much of x^T y is removed in this step).
  const double zeta = (b - a) / (2.0 * c);
  double t;
  if (fabs(zeta) > 1e15) {
    t = 0.5 / zeta;
  } else {
    const float zf = (float)zeta;
    t = (double)(copysignf(1.0f, zf) / (fabsf(zf) + sqrtf(1.0f + zf * zf)));
  }
  const double cs = rsqrt(1.0 + t * t), sn = cs * t;
  double P[NPL], Q[NPL];
#pragma unroll
  for (int q = 0; q < NPL; ++q) {
    const int i = lane + 32 * q;
    P[q] = i < l ? vx[i] : 0.0;
    Q[q] = i < l ? vy[i] : 0.0;
  }
#pragma unroll
  for (int q = 0; q < NPL; ++q) {
    const int i = lane + 32 * q;
    if (i < l) {
      mx[i] = cs * X[q] - sn * Yv[q];
      my[i] = sn * X[q] + cs * Yv[q];
      vx[i] = cs * P[q] - sn * Q[q];
      vy[i] = sn * P[q] + cs * Q[q];
    }
  }
  if (lane == 0) {
    const double cc = cs * cs, ss = sn * sn, cscs = 2.0 * cs * sn * c;
    nrm[x] = cc * a - cscs + ss * b;
    nrm[y] = ss * a + cscs + cc * b;
  }
}

template <int NPL>
__global__ void __launch_bounds__(NPL >= 8 ? 512 : 1024) jacobi_kernel(JacobiArgs a) {
  extern __shared__ __align__(16) double sm[];
  const int l = a.l, bs = a.bs, nb = a.nb;
  const int W = 2 * bs;                 // local column slots: [0,bs) block A, [bs,2bs) block B
  double* Ms = sm;                      // [W][l]
  double* Vs = sm + (size_t)W * l;      // [W][l]
  __shared__ int gcol[64];              // global column of each local slot (-1 = empty)
  __shared__ double nrm[64];
  __shared__ double s_off;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int P = gridDim.x;
  uint32_t* bar = a.bar;

  for (int sweep = 0; sweep < a.max_sweeps; ++sweep) {
    if (tid == 0) s_off = 0.0;
    for (int r = 0; r < nb - 1; ++r) {
      const int pa = rr_player(blockIdx.x, r, nb), pb = rr_player(nb - 1 - blockIdx.x, r, nb);
      if (tid < W) {
        const int blk = tid < bs ? pa : pb;
        const int c = blk * bs + (tid < bs ? tid : tid - bs);
        gcol[tid] = (c < l) ? c : -1;
      }
      __syncthreads();
      for (int idx = tid; idx < W * l; idx += blockDim.x) {
        const int j = idx / l, i = idx - j * l;
        const int c = gcol[j];
        Ms[idx] = c >= 0 ? a.M[i + (int64_t)c * a.ldm] : 0.0;
        Vs[idx] = c >= 0 ? a.V[i + (int64_t)c * a.ldv] : 0.0;
      }
      __syncthreads();
      for (int j = warp; j < W; j += nwarps) {
        const double* mc = Ms + (size_t)j * l;
        double acc = 0.0;
        for (int i = lane; i < l; i += 32) acc = fma(mc[i], mc[i], acc);
        acc = warp_sum(acc);
        if (lane == 0) nrm[j] = acc;
      }
      __syncthreads();
      double off = 0.0;
      if (r == 0) {
        // within-block pairs of both staged blocks, once per sweep (circle method,
        // bs' = bs rounded up to even; pairs touching a phantom slot are skipped)
        const int be = bs + (bs & 1);
        for (int t = 0; t < be - 1; ++t) {
          for (int pr = warp; pr < be; pr += nwarps) {       // be/2 pairs per block
            const int blk = pr < be / 2 ? 0 : 1;
            const int q = pr - blk * (be / 2);
            const int xl = rr_player(q, t, be), yl = rr_player(be - 1 - q, t, be);
            if (xl >= bs || yl >= bs) continue;
            const int x = blk * bs + xl, y = blk * bs + yl;
            if (gcol[x] < 0 || gcol[y] < 0) continue;
            jacobi_pair<NPL>(Ms, Vs, nrm, l, x, y, a.tol, lane, off);
          }
          __syncthreads();
        }
      }
      // cross pairs: bs rounds, warp i pairs A_i with B_{(i+t) mod bs}
      for (int t = 0; t < bs; ++t) {
        for (int i = warp; i < bs; i += nwarps) {
          const int x = i, y = bs + (i + t) % bs;
          if (gcol[x] < 0 || gcol[y] < 0) continue;
          jacobi_pair<NPL>(Ms, Vs, nrm, l, x, y, a.tol, lane, off);
        }
        __syncthreads();
      }
      for (int idx = tid; idx < W * l; idx += blockDim.x) {
        const int j = idx / l, i = idx - j * l;
        const int c = gcol[j];
        if (c >= 0) {
          a.M[i + (int64_t)c * a.ldm] = Ms[idx];
          a.V[i + (int64_t)c * a.ldv] = Vs[idx];
        }
      }
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
  if ((l + 31) / 32 >= 8 && bs > 16) bs = 16;   // register budget of the NPL >= 8 variants
  // keep >= 4 CTAs busy for small l
  while (bs > 4 && (l + bs - 1) / bs < 8) bs /= 2;
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
  void* kern;
  const int npl = (l + 31) / 32;
  if (npl <= 2) kern = (void*)jacobi_kernel<2>;
  else if (npl <= 4) kern = (void*)jacobi_kernel<4>;
  else if (npl <= 8) kern = (void*)jacobi_kernel<8>;
  else if (npl <= 12) kern = (void*)jacobi_kernel<12>;
  else if (npl <= 16) kern = (void*)jacobi_kernel<16>;
  else kern = (void*)jacobi_kernel<32>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
  cudaError_t e = cudaMemsetAsync(bar, 0, 2 * sizeof(uint32_t), st);
  if (e == cudaSuccess) e = cudaMemsetAsync(offmax, 0, sizeof(double) * max_sweeps, st);
  if (e != cudaSuccess) return e;
  const int threads = 32 * (bs < 4 ? 4 : bs);
  void* args[] = {&a};
  e = cudaLaunchCooperativeKernel(kern, dim3(P), dim3(threads), args, smem, st);
  if (e != cudaSuccess) return e;
  jacobi_finish_kernel<<<1, 1024, sizeof(double) * (size_t)l, st>>>(M, ldm, V, ldv, l, sig, U, ldu,
                                                                    Vo, ldvo, order);
  return cudaGetLastError();
}

}  // namespace ffb
