// Small dense SVD (K14): one-sided block Jacobi (Hestenes) on the l x l
// triangular factor of tmp = A P Qhat_1 — replaces LAPACK dgesdd
// (ffsrqr/svd.py:79).  One-sided Jacobi gives singular values to high RELATIVE
// accuracy, which the 1e-10 parity bound needs at the small end of the spectrum.
//
// Cooperative persistent kernel.  Columns are split into nb (even) blocks of bs
// columns; each outer round, CTA p takes one block pair of a round-robin
// tournament (W = 2 bs <= 64 local columns) and
//   1. forms the fresh W x W Gram G = M_W^T M_W on DMMA (64-row chunks staged in
//      shared memory) — the convergence test reads |G_ij| / sqrt(G_ii G_jj);
//   2. diagonalizes the cross-block part with two-sided Jacobi rotations on G
//      (16-32 disjoint pairs per round, one barrier pair per round), accumulating
//      the W x W orthogonal J (within-block pairs once per sweep);
//   3. applies M_W <- M_W J and V_W <- V_W J with DMMA.
// Each visit re-measures G from the actual columns, so rounding in the small
// two-sided iteration never accumulates into the factorization.  A grid barrier
// separates rounds; sweeps stop when max |cos| seen in a sweep <= tol.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "ffb_common.cuh"
#include "ffb_jacobi.cuh"

#include <cooperative_groups.h>
namespace cg = cooperative_groups;

namespace ffb {

namespace {

constexpr int kJThreads = 256;

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

// slot pair k of inner round t: within-block pairs (round-robin over be slots
// of each block) for t < n_within, then cross pairs (k, bs + (k + t') % bs)
constexpr int kBS = 16;   // block size: every inner round pairs all 2 * kBS slots

FFB_DEV void inner_pair(int t, int k, int n_within, int& p, int& q) {
  if (t < n_within) {
    constexpr int np = kBS / 2;
    const int blk = k < np ? 0 : 1, kk = k - blk * np;
    p = blk * kBS + rr_player(kk, t, kBS);
    q = blk * kBS + rr_player(kBS - 1 - kk, t, kBS);
  } else {
    const int tt = (t - n_within) & (kBS - 1);
    p = k;
    q = kBS + ((k + tt) & (kBS - 1));
  }
}

// Jacobi rotation (c, s) of slots (p, q) from the current Gram.  Threshold test
// in fp64 without square roots; the angle t in fp32 with fast intrinsics (t only
// sets how much of x^T y is removed, its accuracy just affects convergence
// speed), c = 1/sqrt(1+t^2) refined to fp64 by two Newton steps so the rotation
// is orthogonal to working precision.  Returns (cc^2, aa*bb) for the caller's
// off-diagonal measure; c = 1, s = 0 when the pair is already orthogonal.
FFB_DEV bool rotation(const double* G, const int* gcol, int p, int q, double tol2, double& c,
                      double& s, double& c2, double& den) {
  c = 1.0;
  s = 0.0;
  c2 = 0.0;
  den = 1.0;
  if (gcol[p] < 0 || gcol[q] < 0) return false;
  const double aa = G[p * 33 + p], bb = G[q * 33 + q], cc = G[p * 33 + q];
  c2 = cc * cc;
  den = aa * bb;
  if (!(c2 > tol2 * den)) return false;
  const float zf = __fdividef((float)(bb - aa), 2.0f * (float)cc);
  double t;
  if (fabsf(zf) < 1e15f) {
    const float az = fabsf(zf), y = fmaf(az, az, 1.0f);
    const float tf = __frcp_rn(az + y * rsqrtf(y));
    t = (double)copysignf(tf, zf);
  } else {
    t = cc / (bb - aa);   // ~ 1 / (2 zeta) for huge |zeta| (or cc underflowed in fp32)
  }
  const double y = fma(t, t, 1.0);
  double r = (double)rsqrtf((float)y);
  r = r * fma(-0.5 * y * r, r, 1.5);
  r = r * fma(-0.5 * y * r, r, 1.5);
  c = r;
  s = r * t;
  return true;
}

}  // namespace

// W (<= 32) local columns: M_W (and V_W when VRES) staged in shared memory
// (l x W, row-major, ld kMW); G and J are W x W.  256 threads.  CLUSTER: the P
// CTAs form one thread-block cluster and rounds are separated by the hardware
// cluster barrier (release/acquire at cluster scope covers the global M, V).
constexpr int kMW = 33;

template <bool CLUSTER>
FFB_DEV void round_barrier(uint32_t* bar, uint32_t P) {
  if (CLUSTER) {
    __syncthreads();
    cg::this_cluster().sync();
  } else {
    grid_barrier(bar, P);
  }
}

// stage the W (=32) local columns of X (rows < l) into S (lpad x kMW) with
// cp.async (zero-fill beyond l / empty slots): every copy of the CTA is in flight
// at once; the caller commits and waits.  Warp w: columns w, w+8, ..; lanes: rows.
FFB_DEV void stage_cols_async(double* S, const double* X, int64_t ldx, const int* gcol, int l,
                              int lpad) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int cc = warp; cc < 32; cc += 8) {
    const int c = gcol[cc];
    const double* src = X + (int64_t)(c < 0 ? 0 : c) * ldx;
    for (int rr = lane; rr < lpad; rr += 32) {
      const bool ok = c >= 0 && rr < l;
      cp_async8(S + rr * kMW + cc, ok ? src + rr : X, ok);
    }
  }
}

// X_W <- S_W J (S: lpad x 32 in smem), written straight to global.  Warp w owns
// row tiles w, w+8, .. (<= 7 for lpad <= 448) x all 4 column tiles: up to 28
// independent DMMA accumulator chains per warp hide the DMMA latency.
FFB_DEV void apply_cols(const double* S, const double* Js, double* X, int64_t ldx,
                        const int* gcol, int l, int lpad) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int fr = lane >> 2, fk = lane & 3;
  const int nrt = lpad >> 3;
  constexpr int kMaxRT = 7;
  for (int g0 = 0; g0 < nrt; g0 += 8 * kMaxRT) {
    double acc[kMaxRT][4][2];
#pragma unroll
    for (int i = 0; i < kMaxRT; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
    for (int k0 = 0; k0 < 32; k0 += 4) {
      double bf[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = Js[(k0 + fk) * 33 + 8 * j + fr];
#pragma unroll
      for (int i = 0; i < kMaxRT; ++i) {
        const int rt = g0 + warp + 8 * i;
        if (rt < nrt) {
          const double af = S[(rt * 8 + fr) * kMW + k0 + fk];
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma_884(acc[i][j][0], acc[i][j][1], af, bf[j]);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < kMaxRT; ++i) {
      const int rt = g0 + warp + 8 * i;
      if (rt >= nrt) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int row = rt * 8 + (lane >> 2), cc = 8 * j + 2 * (lane & 3) + hh;
          const int c = gcol[cc];
          if (c >= 0 && row < l) X[row + (int64_t)c * ldx] = acc[i][j][hh];
        }
    }
  }
}

template <bool CLUSTER, bool VRES>
__global__ void __launch_bounds__(kJThreads, 1) jacobi_kernel(JacobiArgs a) {
  extern __shared__ __align__(16) double sm[];
  const int l = a.l, bs = a.bs, nb = a.nb, W = 2 * bs;   // W <= 32
  const int lpad = (l + 63) & ~63;
  double* Ms = sm;                        // lpad x kMW : M_W (rows >= l zero)
  double* Gs = Ms + (size_t)lpad * kMW;   // 32 x 33
  double* Js = Gs + 32 * 33;              // 32 x 33
  double* Gs2 = Js + 32 * 33;             // ping-pong partners of Gs / Js
  double* Js2 = Gs2 + 32 * 33;
  double* Vs = Js2 + 32 * 33;             // VRES: lpad x kMW ; else 64 x kMW chunk
  __shared__ int gcol[32];
  __shared__ double s_off;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int P = gridDim.x;
  const double tol = a.tol;
  const double tol2 = a.tol * a.tol;

  long long tp[6] = {0, 0, 0, 0, 0, 0};
  long long tc = clock64();
#define JPROF(i)                              \
  if (a.prof && tid == 0) {                   \
    const long long now = clock64();          \
    tp[i] += now - tc;                        \
    tc = now;                                 \
  }
  for (int sweep = 0; sweep < a.max_sweeps; ++sweep) {
    if (tid == 0) s_off = 0.0;
    for (int r = 0; r < nb - 1; ++r) {
      const int pa = rr_player(blockIdx.x, r, nb), pb = rr_player(nb - 1 - blockIdx.x, r, nb);
      if (tid < 32) {
        int c = -1;
        if (tid < W) {
          const int blk = tid < bs ? pa : pb;
          c = blk * bs + (tid < bs ? tid : tid - bs);
          if (c >= l) c = -1;
        }
        gcol[tid] = c;
      }
      __syncthreads();
      stage_cols_async(Ms, a.M, a.ldm, gcol, l, lpad);
      cp_async_commit();
      cp_async_wait<0>();
      __syncthreads();
      JPROF(0)
      // fresh Gram G = M_W^T M_W: warp w sums rows [w*lpad/8, (w+1)*lpad/8) for all
      // 16 output tiles (16 independent DMMA chains), partials reduced through smem
      {
        double* part = VRES ? Vs : Gs;   // 8 x 32 x 33 scratch (VRES: V not staged yet)
        const int fr = lane >> 2, fk = lane & 3;
        double acc[4][4][2];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
        const int kr = lpad >> 3;                 // rows per warp (multiple of 8)
        for (int k0 = warp * kr; k0 < (warp + 1) * kr; k0 += 4) {
          double f[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) f[i] = Ms[(k0 + fk) * kMW + 8 * i + fr];
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) dmma_884(acc[i][j][0], acc[i][j][1], f[i], f[j]);
        }
        if (VRES) {
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
              for (int h = 0; h < 2; ++h)
                part[warp * 32 * 33 + (8 * i + fr) * 33 + 8 * j + 2 * fk + h] = acc[i][j][h];
          __syncthreads();
          for (int t = tid; t < 32 * 32; t += nt) {
            const int r = t >> 5, c = t & 31;
            double sum = 0.0;
#pragma unroll
            for (int w = 0; w < 8; ++w) sum += part[w * 32 * 33 + r * 33 + c];
            Gs[r * 33 + c] = sum;
          }
          __syncthreads();
          // V staging overlaps the inner rotations
          stage_cols_async(Vs, a.V, a.ldv, gcol, l, lpad);
          cp_async_commit();
        } else {
          // no scratch: accumulate warp partials into Gs with fixed-order passes
          for (int t = tid; t < 32 * 32; t += nt) Gs[(t >> 5) * 33 + (t & 31)] = 0.0;
          __syncthreads();
          for (int w = 0; w < 8; ++w) {
            if (warp == w) {
#pragma unroll
              for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j)
#pragma unroll
                  for (int h = 0; h < 2; ++h) Gs[(8 * i + fr) * 33 + 8 * j + 2 * fk + h] += acc[i][j][h];
            }
            __syncthreads();
          }
        }
      }
      for (int t = tid; t < 32 * 32; t += nt) Js[(t >> 5) * 33 + (t & 31)] = ((t >> 5) == (t & 31)) ? 1.0 : 0.0;
      __syncthreads();
      JPROF(1)
      // every round pairs all 32 local slots (16 disjoint pairs); thread (ba, bb2)
      // owns the 2x2 block (pair ba rows, pair bb2 cols) of G and of J.  Lane
      // (x & 15) of each warp computes the rotation of pair x & 15 (no broadcast
      // step; pair ba's rotation comes by shuffle), and the rotated block goes
      // into the other buffer: one barrier per round.
      double offn = 0.0, offd = 1.0;   // running max of G_pq^2 / (G_pp G_qq)
      const int n_within = (r == 0) ? kBS - 1 : 0;
      const int n_cross = a.inner * kBS;
      const int ba = tid >> 4, bb2 = tid & 15;
      const double* Gc = Gs;
      const double* Jc = Js;
      double* Gn = Gs2;
      double* Jn = Js2;
      for (int t = 0; t < n_within + n_cross; ++t) {
        int pa2, qa2, pb2, qb2;
        inner_pair(t, ba, n_within, pa2, qa2);
        inner_pair(t, bb2, n_within, pb2, qb2);
        const double g00 = Gc[pa2 * 33 + pb2], g01 = Gc[pa2 * 33 + qb2];
        const double g10 = Gc[qa2 * 33 + pb2], g11 = Gc[qa2 * 33 + qb2];
        const double j00 = Jc[pa2 * 33 + pb2], j01 = Jc[pa2 * 33 + qb2];
        const double j10 = Jc[qa2 * 33 + pb2], j11 = Jc[qa2 * 33 + qb2];
        double cb, sb, c2b, denb;
        const bool rot = rotation(Gc, gcol, pb2, qb2, tol2, cb, sb, c2b, denb);
        // lane ba of this warp has bb2 == ba: its rotation is pair ba's
        const double ca = __shfl_sync(0xffffffffu, cb, ba);
        const double sa = __shfl_sync(0xffffffffu, sb, ba);
        if (rot && ba == bb2 && c2b * offd > offn * denb) {
          offn = c2b;
          offd = denb;
        }
        // G_blk <- R_a^T G_blk R_b with R = [[c, s], [-s, c]] acting on (p, q)
        const double h00 = cb * g00 - sb * g01, h01 = sb * g00 + cb * g01;   // columns
        const double h10 = cb * g10 - sb * g11, h11 = sb * g10 + cb * g11;
        Gn[pa2 * 33 + pb2] = ca * h00 - sa * h10;
        Gn[pa2 * 33 + qb2] = ca * h01 - sa * h11;
        Gn[qa2 * 33 + pb2] = sa * h00 + ca * h10;
        Gn[qa2 * 33 + qb2] = sa * h01 + ca * h11;
        // J rows (pa, qa) x columns (pb, qb): J <- J R_b (column rotation only)
        Jn[pa2 * 33 + pb2] = cb * j00 - sb * j01;
        Jn[pa2 * 33 + qb2] = sb * j00 + cb * j01;
        Jn[qa2 * 33 + pb2] = cb * j10 - sb * j11;
        Jn[qa2 * 33 + qb2] = sb * j10 + cb * j11;
        __syncthreads();
        const double* tg = Gc;
        Gc = Gn;
        Gn = const_cast<double*>(tg);
        const double* tj = Jc;
        Jc = Jn;
        Jn = const_cast<double*>(tj);
      }
      double off = offn > 0.0 ? sqrt(offn / offd) : 0.0;
      JPROF(2)
      apply_cols(Ms, Jc, a.M, a.ldm, gcol, l, lpad);
      if (VRES) {
        cp_async_wait<0>();
        __syncthreads();
        apply_cols(Vs, Jc, a.V, a.ldv, gcol, l, lpad);
      } else {
        for (int ch = 0; ch < lpad; ch += 64) {
          __syncthreads();
          for (int t = tid; t < 64 * 32; t += nt) {
            const int rr = t & 63, cc = t >> 6;
            const int c = gcol[cc];
            Vs[rr * kMW + cc] = (c >= 0 && ch + rr < l) ? a.V[(ch + rr) + (int64_t)c * a.ldv] : 0.0;
          }
          __syncthreads();
          // reuse apply_cols on one 64-row chunk (rows offset ch)
          const int fr = lane >> 2, fk = lane & 3;
          double acc[4][2];
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[j][0] = acc[j][1] = 0.0;
#pragma unroll
          for (int k0 = 0; k0 < 32; k0 += 4) {
            const double af = Vs[(warp * 8 + fr) * kMW + k0 + fk];
#pragma unroll
            for (int j = 0; j < 4; ++j) dmma_884(acc[j][0], acc[j][1], af, Jc[(k0 + fk) * 33 + 8 * j + fr]);
          }
#pragma unroll
          for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              const int row = ch + warp * 8 + (lane >> 2), cc = 8 * j + 2 * (lane & 3) + hh;
              const int c = gcol[cc];
              if (c >= 0 && row < l) a.V[row + (int64_t)c * a.ldv] = acc[j][hh];
            }
        }
      }
      __syncthreads();
      JPROF(3)
      off = warp_max(off);
      if (lane == 0 && off > 0.0)
        atomicMax(reinterpret_cast<unsigned long long*>(&s_off),
                  (unsigned long long)__double_as_longlong(off));
      __syncthreads();
      if (tid == 0 && s_off > 0.0)
        atomicMax(reinterpret_cast<unsigned long long*>(a.offmax + sweep),
                  (unsigned long long)__double_as_longlong(s_off));
      JPROF(4)
      round_barrier<CLUSTER>(a.bar, P);
      JPROF(5)
    }
    const double om = *((volatile double*)(a.offmax + sweep));
    if (tid == 0 && blockIdx.x == 0) *a.sweeps = sweep + 1;
    if (!(om > tol)) break;
  }
  if (a.prof && tid == 0 && blockIdx.x == 0)
    for (int i = 0; i < 6; ++i) a.prof[i] = tp[i];
#undef JPROF
}

// M <- 2^-e M with 2^e ~ max |M| (exact power-of-two scaling): keeps the Gram
// entries and their fp32 images in range whatever the scale of A.  e -> sweeps[1].
__global__ void jacobi_prescale_kernel(double* M, int64_t ldm, int l, int* sweeps) {
  __shared__ double red[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  double mx = 0.0;
  for (int idx = tid; idx < l * l; idx += blockDim.x) {
    const int j = idx / l, i = idx - j * l;
    mx = fmax(mx, fabs(M[i + (int64_t)j * ldm]));
  }
  mx = warp_max(mx);
  if (lane == 0) red[warp] = mx;
  __syncthreads();
  mx = 0.0;
  for (int w = 0; w < nw; ++w) mx = fmax(mx, red[w]);
  const int e = (mx > 0.0 && isfinite(mx)) ? ilogb(mx) : 0;
  if (tid == 0) sweeps[1] = e;
  if (e == 0) return;
  const double sc = ldexp(1.0, -e);
  for (int idx = tid; idx < l * l; idx += blockDim.x) {
    const int j = idx / l, i = idx - j * l;
    M[i + (int64_t)j * ldm] *= sc;
  }
}

// sigma_j = ||M[:, j]||; rank sort (descending, ties by index); outputs sorted
// sigma, U = M_j / sigma_j (zero column when sigma_j == 0) and V columns.
__global__ void jacobi_finish_kernel(const double* M, int64_t ldm, const double* V, int64_t ldv,
                                     int l, double* sig, double* U, int64_t ldu, double* Vo,
                                     int64_t ldvo, int* order, const int* sweeps) {
  extern __shared__ double nrm[];
  const double unscale = ldexp(1.0, sweeps[1]);
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
    sig[rank] = sj * unscale;
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
  (void)l;
  return 16;   // every inner round pairs all 32 staged slots (empty slots rotate trivially)
}

cudaError_t launch_jacobi_svd(cudaStream_t st, int sms, double* M, int64_t ldm, double* V,
                              int64_t ldv, int l, double* sig, double* U, int64_t ldu, double* Vo,
                              int64_t ldvo, uint32_t* bar, double* offmax, int* sweeps, int* order,
                              int max_sweeps) {
  (void)sms;
  const int bs = jacobi_block_size(l);
  int nb = (l + bs - 1) / bs;
  if (nb % 2) ++nb;
  if (nb < 2) nb = 2;
  const int P = nb / 2;
  int inner = 1;
  if (const char* e = getenv("FFB_JACOBI_INNER")) inner = atoi(e);
  if (inner < 1) inner = 1;
  static long long* prof = nullptr;
  if (getenv("FFB_JACOBI_PROF") && !prof) cudaMallocManaged(&prof, 8 * sizeof(long long));
  JacobiArgs a{M, ldm, V, ldv, l, bs, nb, 1e-15 * sqrt((double)l), max_sweeps, bar, offmax, sweeps, inner, prof};
  const size_t lpad = (size_t)((l + 63) & ~63);
  const size_t fixed = sizeof(double) * (lpad * kMW + 4 * 32 * 33);
  // V region: V_W when resident (>= 8 x 32 x 33 doubles, it doubles as Gram scratch)
  const size_t vreg = sizeof(double) * (lpad > 256 ? lpad : 256) * kMW;
  const bool vres = fixed + vreg <= 220 * 1024;
  const size_t smem = vres ? fixed + vreg : fixed + sizeof(double) * 64 * kMW;
  if (smem > 220 * 1024) return cudaErrorInvalidValue;   // l > ~800 not supported
  const bool cluster = P <= 16 && getenv("FFB_JACOBI_NOCLUSTER") == nullptr;
  void* kern = cluster ? (vres ? (void*)jacobi_kernel<true, true> : (void*)jacobi_kernel<true, false>)
                       : (vres ? (void*)jacobi_kernel<false, true> : (void*)jacobi_kernel<false, false>);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaError_t e = cudaMemsetAsync(bar, 0, 2 * sizeof(uint32_t), st);
  if (e == cudaSuccess) e = cudaMemsetAsync(offmax, 0, sizeof(double) * max_sweeps, st);
  if (e != cudaSuccess) return e;
  jacobi_prescale_kernel<<<1, 1024, 0, st>>>(M, ldm, l, sweeps);
  void* args[] = {&a};
  if (cluster) {
    if (P > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(P);
    cfg.blockDim = dim3(kJThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = P;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelExC(&cfg, kern, args);
  } else {
    e = cudaLaunchCooperativeKernel(kern, dim3(P), dim3(kJThreads), args, smem, st);
  }
  if (e != cudaSuccess) return e;
  jacobi_finish_kernel<<<1, 1024, sizeof(double) * (size_t)l, st>>>(M, ldm, V, ldv, l, sig, U, ldu,
                                                                    Vo, ldvo, order, sweeps);
  if (prof) {
    cudaStreamSynchronize(st);
    fprintf(stderr, "jacobi phases (cycles, CTA0): stage %lld gram %lld inner %lld apply %lld off %lld barrier %lld\n",
            prof[0], prof[1], prof[2], prof[3], prof[4], prof[5]);
  }
  return cudaGetLastError();
}

}  // namespace ffb
