// Non-GEMM kernels of the Flip-Flop SRQR engine (sm_100a).
//
// Reference semantics cited per kernel; see DESIGN.md for the data layout:
// A, B (sketch), R, WT are kept in ORIGINAL column order and an arrangement
// array arr[pos] = column (with its inverse pos[column]) replaces the
// reference's physical reorders (ffsrqr/sketch.py:70-72,120-121).
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "ffb_common.cuh"
#include "ffb_kernels.cuh"
#include "ffb_pivot_dev.cuh"
#include "ffb_tile64.cuh"

namespace ffb {

#define FFB_LAUNCH_CHECK() return cudaGetLastError()

FFB_DEV void st_release_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
FFB_DEV uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
FFB_DEV uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

static inline unsigned nblk(int64_t work, int per) {
  int64_t b = (work + per - 1) / per;
  if (b < 1) b = 1;
  if (b > 2147483647LL) b = 2147483647LL;
  return (unsigned)b;
}

// ----------------------------------------------------------------- basics

__global__ void colsq_kernel(const double* __restrict__ A, int64_t lda, int64_t m, int64_t n,
                             double* __restrict__ colsq) {
  const int lane = threadIdx.x & 31;
  const int64_t col = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (col >= n) return;
  const double* a = A + col * lda;
  double s0 = 0.0, s1 = 0.0;
  int64_t i = lane;
  for (; i + 32 < m; i += 64) {
    const double x = a[i], y = a[i + 32];
    s0 = fma(x, x, s0);
    s1 = fma(y, y, s1);
  }
  if (i < m) s0 = fma(a[i], a[i], s0);
  const double s = warp_sum(s0 + s1);
  if (lane == 0) colsq[col] = s;
}

cudaError_t launch_colsq(cudaStream_t st, const double* A, int64_t lda, int64_t m, int64_t n,
                         double* colsq) {
  colsq_kernel<<<nblk(n, 8), 256, 0, st>>>(A, lda, m, n, colsq);
  FFB_LAUNCH_CHECK();
}

// Row-major A (A(i, j) = A[i * lda + j]): thread per column, coalesced along
// rows; kColsqSplit row slabs write partial sums that a second pass adds in
// slab order (deterministic).
constexpr int kColsqSplit = 16;
__global__ void colsq_rm_kernel(const double* __restrict__ A, int64_t lda, int64_t m, int64_t n,
                                double* __restrict__ part) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int64_t per = (m + kColsqSplit - 1) / kColsqSplit;
  const int64_t i0 = blockIdx.y * per, i1 = i0 + per < m ? i0 + per : m;
  double s0 = 0.0, s1 = 0.0;
  int64_t i = i0;
  for (; i + 1 < i1; i += 2) {
    const double x = A[i * lda + j], y = A[(i + 1) * lda + j];
    s0 = fma(x, x, s0);
    s1 = fma(y, y, s1);
  }
  if (i < i1) s0 = fma(A[i * lda + j], A[i * lda + j], s0);
  part[blockIdx.y * n + j] = s0 + s1;
}

__global__ void colsq_rm_sum_kernel(const double* __restrict__ part, int64_t n, double* colsq) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  double s = 0.0;
  for (int q = 0; q < kColsqSplit; ++q) s += part[q * n + j];
  colsq[j] = s;
}

size_t colsq_rm_part_doubles(int64_t n) { return (size_t)kColsqSplit * (size_t)n; }

cudaError_t launch_colsq_rm(cudaStream_t st, const double* A, int64_t lda, int64_t m, int64_t n,
                            double* part, double* colsq) {
  colsq_rm_kernel<<<dim3(nblk(n, 256), kColsqSplit), 256, 0, st>>>(A, lda, m, n, part);
  colsq_rm_sum_kernel<<<nblk(n, 256), 256, 0, st>>>(part, n, colsq);
  FFB_LAUNCH_CHECK();
}

__global__ void iota2_kernel(int64_t* arr, int64_t* pos, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    arr[i] = i;
    pos[i] = i;
  }
}

cudaError_t launch_iota2(cudaStream_t st, int64_t* arr, int64_t* pos, int64_t n) {
  iota2_kernel<<<nblk(n, 256) > 1024 ? 1024 : nblk(n, 256), 256, 0, st>>>(arr, pos, n);
  FFB_LAUNCH_CHECK();
}

// ------------------------------------------------ sketch QRCP pivots (K2)
//
// bb steps of Householder QRCP on a working copy of the sketch's trailing
// columns (positions >= j0), returning only the swap-history arrangement —
// ffsrqr/sketch.py:62-67 -> ffsrqr/_kernels_numba.py:15-94.  Cooperative
// persistent kernel: CTA g owns original columns [g*cpc, (g+1)*cpc) in shared
// memory (or an L2-resident global slab when they do not fit).  Each step:
// local candidate -> publish (r, position, column data) -> one all-to-all flag
// wait -> every CTA picks the same global winner (largest r, ties to the lowest
// position) and computes the same reflector -> local update + norm downdate
// with the 1e-8 guard recompute.

// top-2 candidate (r, position); better = larger r, ties -> lower position
struct Cand2 {
  double r1;
  int64_t p1;
  double r2;
  int64_t p2;
};

FFB_DEV void cand_push(Cand2& c, double r, int64_t p) {
  if (cand_better(r, p, c.r1, c.p1)) {
    c.r2 = c.r1;
    c.p2 = c.p1;
    c.r1 = r;
    c.p1 = p;
  } else if (cand_better(r, p, c.r2, c.p2)) {
    c.r2 = r;
    c.p2 = p;
  }
}

FFB_DEV Cand2 cand_merge(Cand2 a, const Cand2& b) {
  cand_push(a, b.r1, b.p1);
  cand_push(a, b.r2, b.p2);
  return a;
}

FFB_DEV Cand2 cand_shfl(const Cand2& c, int off) {
  Cand2 o;
  o.r1 = __shfl_xor_sync(0xffffffffu, c.r1, off);
  o.p1 = __shfl_xor_sync(0xffffffffu, c.p1, off);
  o.r2 = __shfl_xor_sync(0xffffffffu, c.r2, off);
  o.p2 = __shfl_xor_sync(0xffffffffu, c.p2, off);
  return o;
}

FFB_DEV Cand2 warp_top2(Cand2 c) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c = cand_merge(c, cand_shfl(c, o));
  return c;
}

// Column storage: column-major per column with padded stride sP (sP % 16 == 4),
// 4 threads per column (interleaved rows).  kGroups column groups per CTA.
constexpr int kPivThreads = 256;
constexpr int kPivGroups = kPivThreads / 4;
constexpr int kPivMaxK = 5;   // CTAs per lane in the header exchange (G <= 160)

// RQ > 0: every column group owns at most one column and keeps its rows
// (sub + 4q, q < RQ) in registers; shared memory gets a write-through copy that
// the publish step reads.  RQ == 0: generic shared/global-memory loop with the
// rows of a column loaded to registers (s <= 128).  RQ == -1: generic loop
// straight on shared/global memory (any s).  RQ == -2 (global memory, s <= 48,
// many columns per CTA, e.g. a 400 x 160000 unfolding's sketch): one THREAD per
// column, W stored row-major ([s][cpc]) so a warp's loads of one sketch row are
// coalesced and every column's s loads are in flight at once.  XQ: winner-column
// rows per lane of the reflector warp (s <= 32 XQ).
template <bool SMEM, int RQ, int XQ>
__global__ void __launch_bounds__(kPivThreads, 1) pivots_kernel(PivotArgs a) {
  extern __shared__ __align__(16) double sm[];
  const int s = a.s, cpc = a.cpc, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int sP = a.sP;
  const int grp = tid >> 2, sub = tid & 3;
  const unsigned gmask = 0xFu << (lane & 28);   // the 4 lanes sharing a column
  const int64_t c0 = (int64_t)blockIdx.x * cpc;
  int64_t ncl = a.n - c0;
  if (ncl > cpc) ncl = cpc;
  if (ncl < 0) ncl = 0;
  const int nc = (int)ncl;
  double* W = SMEM ? sm : a.work + (size_t)blockIdx.x * sP * cpc;   // [cpc][sP] ([s][cpc] for RQ == -2)
  constexpr bool kRowMajor = RQ == -2;
  constexpr int kS2 = 48;   // RQ == -2: max sketch rows (registers)
  // element (i, c) of the CTA's column slab
  auto widx = [&](int c, int i) -> size_t { return kRowMajor ? (size_t)i * cpc + c : (size_t)c * sP + i; };
  double* base = SMEM ? sm + (size_t)sP * cpc : sm;
  double* r = base;
  double* r0 = r + cpc;
  int64_t* pp = reinterpret_cast<int64_t*>(r0 + cpc);
  double* vv = reinterpret_cast<double*>(pp + cpc);     // reflector v (s)
  Cand2* wc = reinterpret_cast<Cand2*>(vv + ((s + 1) & ~1));   // per-warp top-2 [8]
  __shared__ double s_tau;
  __shared__ int64_t s_wpos;
  __shared__ double s_hr[kPivThreads / 32];    // spread exchange: the warps' local winners
  __shared__ int64_t s_hp[kPivThreads / 32];
  __shared__ double s_xst[128];                // owner warp: the candidate column, rows by lane

  for (int idx = tid; idx < s * nc; idx += kPivThreads) {
    const int c = idx / s, i = idx - c * s;
    W[widx(c, i)] = a.B[i + (c0 + c) * a.ldb];
  }
  for (int c = tid; c < nc; c += kPivThreads) pp[c] = a.pos[c0 + c];
  __syncthreads();
  double x[RQ > 0 ? RQ : 1];
  (void)x;
  if constexpr (RQ > 0) {
#pragma unroll
    for (int q = 0; q < RQ; ++q) {
      const int i = sub + 4 * q;
      x[q] = (grp < nc && i < s) ? W[(size_t)grp * sP + i] : 0.0;
    }
  }
  // initial norms and local top-2 over positions >= j0
  if constexpr (kRowMajor) {
    Cand2 cd{-1.0, -1, -1.0, -1};
    for (int c = tid; c < nc; c += kPivThreads) {
      double t0 = 0.0, t1 = 0.0;
      int i = 0;
      for (; i + 1 < s; i += 2) {
        const double u = W[widx(c, i)], v = W[widx(c, i + 1)];
        t0 = fma(u, u, t0);
        t1 = fma(v, v, t1);
      }
      if (i < s) t0 = fma(W[widx(c, i)], W[widx(c, i)], t0);
      const double t = t0 + t1;
      r[c] = t;
      r0[c] = t;
      if (pp[c] >= a.j0) cand_push(cd, t, pp[c]);
    }
    cd = warp_top2(cd);
    if (lane == 0) wc[warp] = cd;
  } else {
    Cand2 cd{-1.0, -1, -1.0, -1};
    for (int c = grp; c < nc; c += kPivGroups) {
      const double* col = W + (size_t)c * sP;
      double t = 0.0;
      for (int i = sub; i < s; i += 4) t = fma(col[i], col[i], t);
      t += __shfl_xor_sync(gmask, t, 1);
      t += __shfl_xor_sync(gmask, t, 2);
      if (sub == 0) {
        r[c] = t;
        r0[c] = t;
      }
      if (pp[c] >= a.j0) cand_push(cd, t, pp[c]);
    }
    cd = warp_top2(cd);
    if (lane == 0) wc[warp] = cd;
  }
  __syncthreads();

  long long tp[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long tlast = clock64();
#define PPROF(i)                        \
  if (a.prof && tid == 0) {             \
    const long long tn = clock64();     \
    tp[i] += tn - tlast;                \
    tlast = tn;                         \
  }
  for (int j = 0; j < a.bb; ++j) {
    const int64_t P = a.j0 + j;
    const int par = j & 1;
    // Register-resident columns without gap tracing: the exchange is spread over
    // the CTA instead of running in warp 0 alone.  Every warp derives the CTA's
    // candidate; the warp that owns the candidate column publishes the header
    // and builds the column's reflector (ffsrqr/qr.py:21-43) straight from the
    // owning threads' registers, publishing (tau, v) while the other seven warps
    // poll the headers of the G CTAs (one per lane) and fetch THEIR best CTA's
    // reflector right away; the warp that holds the global winner's hands it to
    // the CTA.  The reflector arithmetic is off the path between the global pick
    // and the update, and the winner's load no longer waits for the pick.
    bool spread = false;
    if constexpr ((RQ >= 0 && SMEM) || RQ == -2) spread = a.gap == nullptr && s <= 32 * XQ;
    if (spread) {
      const uint32_t tag = (uint32_t)(j + 1);
      unsigned long long* base = a.rec + (size_t)par * a.G * a.recw;
      Cand2 cd = lane < (kPivThreads / 32) ? wc[lane] : Cand2{-1.0, -1, -1.0, -1};
      const int64_t wp = cd.p1;              // this lane's warp candidate (lane < 8)
      warp_best(cd.r1, cd.p1);
      // the warp that owns the CTA's candidate column builds that column's
      // reflector while the other warps poll: if the candidate wins globally its
      // v is already on its way to L2 when the pollers ask for it
      const int ow = (int)__ffs(__ballot_sync(0xffffffffu, lane < (kPivThreads / 32) && cd.p1 >= 0 && wp == cd.p1)) - 1;
      unsigned long long* rec = base + (size_t)blockIdx.x * a.recw;
      double lr = -1.0;
      int64_t lp = -1;
      double xv[XQ];
      double ltau = 0.0;
#pragma unroll
      for (int q = 0; q < XQ; ++q) xv[q] = 0.0;
      if (warp == (ow >= 0 ? ow : 0)) {
        // ---- candidate header first, then (owner warp) the reflector of the column
        if (lane == 0)
          st_ll2(rec, ll_pack((uint32_t)__double2loint(cd.r1), tag), ll_pack((uint32_t)__double2hiint(cd.r1), tag));
        if (lane == 1) st_ll2(rec + 2, ll_pack((uint32_t)(int32_t)cd.p1, tag), ll_pack(0u, tag));
        if (ow >= 0) {
          int cl = 0;   // RQ <= 0: the candidate column, read in place through widx
          if constexpr (RQ > 0) {
            if (grp < nc && pp[grp] == cd.p1) {
#pragma unroll
              for (int q = 0; q < RQ; ++q) {
                const int i = sub + 4 * q;
                if (i < s) s_xst[i] = x[q];
              }
            }
          } else {
            // columns in shared / global memory (more than 64 per CTA): the candidate
            // is one of this warp's columns (grp, grp + 64, .. or, one thread per
            // column, tid, tid + 256, ..)
            int c1 = -1;
            for (int c = kRowMajor ? tid : grp; c < nc; c += kRowMajor ? kPivThreads : kPivGroups)
              if (pp[c] == cd.p1) c1 = c;
            c1 = (int)__reduce_max_sync(0xffffffffu, (unsigned)(c1 + 1)) - 1;
            cl = c1 >= 0 ? c1 : 0;
          }
          __syncwarp();
          double xr[XQ];
#pragma unroll
          for (int q = 0; q < XQ; ++q) {
            const int i = lane + 32 * q;
            if constexpr (RQ > 0) xr[q] = (i >= j && i < s) ? s_xst[i] : 0.0;
            else xr[q] = (i >= j && i < s) ? W[widx(cl, i)] : 0.0;
          }
          __syncwarp();
          double tsq = 0.0;
#pragma unroll
          for (int q = 0; q < XQ; ++q) {
            const int i = lane + 32 * q;
            if (i > j && i < s) tsq = fma(xr[q], xr[q], tsq);
          }
          tsq = warp_sum(tsq);
          double xsel = 0.0;
#pragma unroll
          for (int q = 0; q < XQ; ++q) xsel = sel_f64(q == (j >> 5), xr[q], xsel);
          const double x0 = __shfl_sync(0xffffffffu, xsel, j & 31);
          double tau = 0.0, div = 1.0;
          if (tsq != 0.0) {
            const double nrm = sqrt(x0 * x0 + tsq);
            const double alpha = x0 == 0.0 ? nrm : -copysign(nrm, x0);
            div = x0 - alpha;
            tau = (alpha - x0) / alpha;
          }
#pragma unroll
          for (int q = 0; q < XQ; ++q) {
            const int i = lane + 32 * q;
            if (i >= j && i < s) {
              const double v = (i == j) ? 1.0 : (tau != 0.0 ? xr[q] / div : 0.0);
              st_ll2(rec + 8 + 2 * i, ll_pack((uint32_t)__double2loint(v), tag),
                     ll_pack((uint32_t)__double2hiint(v), tag));
            }
          }
          if (lane == 2)
            st_ll2(rec + 4, ll_pack((uint32_t)__double2loint(tau), tag), ll_pack((uint32_t)__double2hiint(tau), tag));
        }
        PPROF(0)
      }
      if (ow < 0 || warp != ow) {
        // ---- pollers: warp index among the np polling warps; lane k polls CTA idx + np k
        const int np = ow >= 0 ? kPivThreads / 32 - 1 : kPivThreads / 32;
        const int idx = (ow >= 0 && warp > ow) ? warp - 1 : warp;
        const int myc = idx + np * lane;
        unsigned long long h0 = 0, h1 = 0, h2 = 0, h3 = 0;
        bool need = myc < a.G;
        do {
          if (need) {
            const unsigned long long* rc = base + (size_t)myc * a.recw;
            ld_ll2(rc, h0, h1);
            ld_ll2(rc + 2, h2, h3);
            if (ll_tag(h0) == tag && ll_tag(h1) == tag && ll_tag(h2) == tag && ll_tag(h3) == tag) need = false;
          }
        } while (__any_sync(0xffffffffu, need));
        PPROF(1)
        if (myc < a.G) {
          lr = __hiloint2double((int)ll_data(h1), (int)ll_data(h0));
          lp = (int64_t)(int32_t)ll_data(h2);
        }
        const int64_t mine = lp;
        warp_best(lr, lp);
        const int wcta = (int)__reduce_max_sync(0xffffffffu, (lp >= 0 && mine == lp) ? (unsigned)(myc + 1) : 0u) - 1;
        // v rows j.. and tau of the local winner (its owner warp may still be at work)
        if (wcta >= 0) {
          const unsigned long long* wrec = base + (size_t)wcta * a.recw;
          unsigned long long xw[XQ][2], t0 = 0, t1 = 0;
          unsigned xneed = 1u << XQ;
#pragma unroll
          for (int q = 0; q < XQ; ++q) {
            const int i = lane + 32 * q;
            if (i >= j && i < s) xneed |= 1u << q;
            xw[q][0] = xw[q][1] = 0ull;
          }
          do {
            if (xneed & (1u << XQ)) ld_ll2(wrec + 4, t0, t1);
#pragma unroll
            for (int q = 0; q < XQ; ++q)
              if (xneed & (1u << q)) ld_ll2(wrec + 8 + 2 * (lane + 32 * q), xw[q][0], xw[q][1]);
            if ((xneed & (1u << XQ)) && ll_tag(t0) == tag && ll_tag(t1) == tag) xneed &= ~(1u << XQ);
#pragma unroll
            for (int q = 0; q < XQ; ++q)
              if ((xneed & (1u << q)) && ll_tag(xw[q][0]) == tag && ll_tag(xw[q][1]) == tag)
                xneed &= ~(1u << q);
          } while (__any_sync(0xffffffffu, xneed != 0));
          ltau = __hiloint2double((int)ll_data(t1), (int)ll_data(t0));
#pragma unroll
          for (int q = 0; q < XQ; ++q) {
            const int i = lane + 32 * q;
            xv[q] = (i >= j && i < s) ? __hiloint2double((int)ll_data(xw[q][1]), (int)ll_data(xw[q][0])) : 0.0;
          }
        }
      }
      if (lane == 0) {
        s_hr[warp] = lr;
        s_hp[warp] = lp;
      }
      __syncthreads();
      PPROF(2)
      // global pick over the polling warps' local winners (every warp, identical)
      double rg = lane < (kPivThreads / 32) ? s_hr[lane] : -1.0;
      int64_t pg = lane < (kPivThreads / 32) ? s_hp[lane] : -1;
      warp_best(rg, pg);
      if (pg >= 0 ? (lp == pg) : (warp == 0)) {
        // the warp holding the winner's reflector hands it to the CTA
        const double tau = pg >= 0 ? ltau : 0.0;
#pragma unroll
        for (int q = 0; q < XQ; ++q) {
          const int i = lane + 32 * q;
          if (i < s) vv[i] = pg >= 0 ? xv[q] : (i == j ? 1.0 : 0.0);
        }
        if (lane == 0) {
          s_tau = tau;
          s_wpos = pg >= 0 ? pg : P;
          if (blockIdx.x == 0) a.hist[j] = pg >= 0 ? pg : P;
        }
      }
      PPROF(3)
    } else if (warp == 0) {
      // ---- local candidate -> publish (tagged LL words, no fences) -> global
      // pick -> reflector, all in warp 0
      const uint32_t tag = (uint32_t)(j + 1);
      unsigned long long* base = a.rec + (size_t)par * a.G * a.recw;
      Cand2 cd = lane < (kPivThreads / 32) ? wc[lane] : Cand2{-1.0, -1, -1.0, -1};
      if (a.gap) {
        cd = warp_top2(cd);
      } else {
        warp_best(cd.r1, cd.p1);
        cd.r2 = -1.0;
        cd.p2 = -1;
      }
      {
        unsigned long long* rec = base + (size_t)blockIdx.x * a.recw;
        if (cd.p1 >= 0) {
          // local column holding position cd.p1 (positions are unique)
          int cl = -1;
          for (int c = lane; c < nc; c += 32)
            if (pp[c] == cd.p1) cl = c;
          cl = (int)__reduce_max_sync(0xffffffffu, (unsigned)(cl + 1)) - 1;
          for (int i = j + lane; i < s; i += 32) {
            const double x = W[widx(cl, i)];
            st_ll2(rec + 8 + 2 * i, ll_pack((uint32_t)__double2loint(x), tag),
                   ll_pack((uint32_t)__double2hiint(x), tag));
          }
        }
        if (lane == 0)
          st_ll2(rec, ll_pack((uint32_t)__double2loint(cd.r1), tag),
                 ll_pack((uint32_t)__double2hiint(cd.r1), tag));
        if (lane == 1)
          st_ll2(rec + 2, ll_pack((uint32_t)(int32_t)cd.p1, tag), ll_pack((uint32_t)(int32_t)cd.p2, tag));
        if (lane == 2 && a.gap)
          st_ll2(rec + 4, ll_pack((uint32_t)__double2loint(cd.r2), tag),
                 ll_pack((uint32_t)__double2hiint(cd.r2), tag));
      }
      PPROF(0)
      // every CTA's header: lane handles CTAs lane + 32k; all loads in flight at once
      unsigned long long h[kPivMaxK][4];
      unsigned need = 0;
#pragma unroll
      for (int k = 0; k < kPivMaxK; ++k)
        if (lane + 32 * k < a.G) need |= 1u << k;
      do {
#pragma unroll
        for (int k = 0; k < kPivMaxK; ++k)
          if (need & (1u << k)) {
            const unsigned long long* rc = base + (size_t)(lane + 32 * k) * a.recw;
            ld_ll2(rc, h[k][0], h[k][1]);
            ld_ll2(rc + 2, h[k][2], h[k][3]);
          }
#pragma unroll
        for (int k = 0; k < kPivMaxK; ++k)
          if ((need & (1u << k)) && ll_tag(h[k][0]) == tag && ll_tag(h[k][1]) == tag &&
              ll_tag(h[k][2]) == tag && ll_tag(h[k][3]) == tag)
            need &= ~(1u << k);
      } while (__any_sync(0xffffffffu, need != 0));
      PPROF(1)
      // global pick: largest r, ties to the lowest position; winner CTA tracked
      Cand2 g{-1.0, -1, -1.0, -1};
      int bc = -1;
#pragma unroll
      for (int k = 0; k < kPivMaxK; ++k)
        if (lane + 32 * k < a.G) {
          const double rr = __hiloint2double((int)ll_data(h[k][1]), (int)ll_data(h[k][0]));
          const int64_t pq = (int64_t)(int32_t)ll_data(h[k][2]);
          if (cand_better(rr, pq, g.r1, g.p1)) bc = lane + 32 * k;
          cand_push(g, rr, pq);
        }
      const int64_t mine = g.p1;
      Cand2 gw = g;
      if (a.gap) {
        gw = warp_top2(g);
      } else {
        warp_best(gw.r1, gw.p1);
        gw.p2 = -1;
      }
      const bool holder = gw.p1 >= 0 && mine == gw.p1;
      const int wc_cta = (int)__reduce_max_sync(0xffffffffu, holder ? (unsigned)(bc + 1) : 0u) - 1;
      double second = (gw.p2 >= 0) ? gw.r2 : -1.0;
      if (a.gap && wc_cta >= 0) {
        // runner-up inside the winner CTA (gap tracing only: one more load)
        const unsigned long long* rc = base + (size_t)wc_cta * a.recw;
        unsigned long long w2, w3, w4, w5;
        do {
          ld_ll2(rc + 2, w2, w3);
          ld_ll2(rc + 4, w4, w5);
        } while (ll_tag(w3) != tag || ll_tag(w4) != tag || ll_tag(w5) != tag);
        if ((int32_t)ll_data(w3) >= 0)
          second = fmax(second, __hiloint2double((int)ll_data(w5), (int)ll_data(w4)));
      }
      const int64_t wpos = gw.p1 >= 0 ? gw.p1 : P;
      PPROF(2)
      // winner column rows j..s-1 -> reflector (ffsrqr/qr.py:21-43)
      double xv[XQ];
      {
        const unsigned long long* wrec = base + (size_t)(wc_cta >= 0 ? wc_cta : 0) * a.recw + 8;
        unsigned long long xw[XQ][2];
        unsigned xneed = 0;
#pragma unroll
        for (int q = 0; q < XQ; ++q) {
          const int i = lane + 32 * q;
          if (i >= j && i < s && wc_cta >= 0) xneed |= 1u << q;
          xw[q][0] = xw[q][1] = 0ull;
        }
        do {
#pragma unroll
          for (int q = 0; q < XQ; ++q)
            if (xneed & (1u << q)) ld_ll2(wrec + 2 * (lane + 32 * q), xw[q][0], xw[q][1]);
#pragma unroll
          for (int q = 0; q < XQ; ++q)
            if ((xneed & (1u << q)) && ll_tag(xw[q][0]) == tag && ll_tag(xw[q][1]) == tag)
              xneed &= ~(1u << q);
        } while (__any_sync(0xffffffffu, xneed != 0));
#pragma unroll
        for (int q = 0; q < XQ; ++q) {
          const int i = lane + 32 * q;
          xv[q] = (i >= j && i < s && wc_cta >= 0)
                      ? __hiloint2double((int)ll_data(xw[q][1]), (int)ll_data(xw[q][0]))
                      : 0.0;
        }
      }
      double tsq = 0.0;
#pragma unroll
      for (int q = 0; q < XQ; ++q) {
        const int i = lane + 32 * q;
        if (i > j && i < s) tsq = fma(xv[q], xv[q], tsq);
      }
      tsq = warp_sum(tsq);
      double xsel = 0.0;
#pragma unroll
      for (int q = 0; q < XQ; ++q) xsel = sel_f64(q == (j >> 5), xv[q], xsel);
      const double x0 = __shfl_sync(0xffffffffu, xsel, j & 31);
      double tau = 0.0, div = 1.0;
      if (tsq != 0.0) {
        const double nrm = sqrt(x0 * x0 + tsq);
        const double alpha = x0 == 0.0 ? nrm : -copysign(nrm, x0);
        div = x0 - alpha;
        tau = (alpha - x0) / alpha;
      }
#pragma unroll
      for (int q = 0; q < XQ; ++q) {
        const int i = lane + 32 * q;
        if (i < s) vv[i] = (i == j) ? 1.0 : (i > j && tau != 0.0 ? xv[q] / div : 0.0);
      }
      if (lane == 0) {
        s_tau = tau;
        s_wpos = wpos;
        if (blockIdx.x == 0) {
          // arr (the inverse of pos) is rebuilt from pos after the loop: no global
          // loads on CTA 0's per-step critical path
          a.hist[j] = wpos;
          if (a.gap) a.gap[j] = (gw.r1 > 0.0 && second >= 0.0) ? (gw.r1 - second) / gw.r1 : 1.0;
        }
      }
      PPROF(3)
    }
    __syncthreads();
    PPROF(4)
    // ---- all threads: swap bookkeeping, reflector application, downdate
    const double tau = s_tau;
    const int64_t wpos = s_wpos;
    Cand2 cd{-1.0, -1, -1.0, -1};
    if constexpr (RQ > 0) {
      const int c = grp;
      if (c < nc) {
        int64_t p = pp[c];
        if (p == wpos) p = P;
        else if (p == P) p = wpos;
        if (sub == 0) pp[c] = p;
        if (p > P) {
          double* col = W + (size_t)c * sP;
          if (tau != 0.0) {
            double w0 = 0.0, w1 = 0.0;
#pragma unroll
            for (int q = 0; q < RQ; ++q) {
              const int i = sub + 4 * q;
              if (i >= j && i < s) {
                if (q & 1) w1 = fma(vv[i], x[q], w1);
                else w0 = fma(vv[i], x[q], w0);
              }
            }
            double wsum = w0 + w1;
            wsum += __shfl_xor_sync(gmask, wsum, 1);
            wsum += __shfl_xor_sync(gmask, wsum, 2);
            const double wt = wsum * tau;
#pragma unroll
            for (int q = 0; q < RQ; ++q) {
              const int i = sub + 4 * q;
              if (i >= j && i < s) {
                x[q] = fma(-vv[i], wt, x[q]);
                if (!spread) col[i] = x[q];   // the warp-0 publish reads the column from shared memory
              }
            }
          }
          double xj = 0.0;
#pragma unroll
          for (int q = 0; q < RQ; ++q) mov_if_f64(xj, q == (j >> 2), x[q]);
          const double rj = __shfl_sync(gmask, xj, (lane & ~3) | (j & 3));
          double rr = r[c] - rj * rj;
          if (rr < 1e-8 * r0[c] || rr < 0.0) {
            double t = 0.0;
#pragma unroll
            for (int q = 0; q < RQ; ++q) {
              const int i = sub + 4 * q;
              if (i > j && i < s) t = fma(x[q], x[q], t);
            }
            t += __shfl_xor_sync(gmask, t, 1);
            t += __shfl_xor_sync(gmask, t, 2);
            rr = t > 0.0 ? t : 0.0;
          }
          if (sub == 0) r[c] = rr;
          cand_push(cd, rr, p);
        }
      }
    } else if constexpr (kRowMajor) {
      for (int c = tid; c < nc; c += kPivThreads) {
        int64_t p = pp[c];
        if (p == wpos) p = P;
        else if (p == P) p = wpos;
        pp[c] = p;
        if (p <= P) continue;
        double xr[kS2];
#pragma unroll
        for (int i = 0; i < kS2; ++i) xr[i] = (i >= j && i < s) ? W[widx(c, i)] : 0.0;
        if (tau != 0.0) {
          double w0 = 0.0, w1 = 0.0;
#pragma unroll
          for (int i = 0; i < kS2; ++i)
            if (i >= j && i < s) {
              if (i & 1) w1 = fma(vv[i], xr[i], w1);
              else w0 = fma(vv[i], xr[i], w0);
            }
          const double wt = (w0 + w1) * tau;
#pragma unroll
          for (int i = 0; i < kS2; ++i)
            if (i >= j && i < s) {
              xr[i] = fma(-vv[i], wt, xr[i]);
              W[widx(c, i)] = xr[i];
            }
        }
        double rj = 0.0;
#pragma unroll
        for (int i = 0; i < kS2; ++i) rj = sel_f64(i == j, xr[i], rj);
        double rr = r[c] - rj * rj;
        if (rr < 1e-8 * r0[c] || rr < 0.0) {
          double t = 0.0;
#pragma unroll
          for (int i = 0; i < kS2; ++i)
            if (i > j && i < s) t = fma(xr[i], xr[i], t);
          rr = t > 0.0 ? t : 0.0;
        }
        r[c] = rr;
        cand_push(cd, rr, p);
      }
    } else if constexpr (RQ < 0) {
      for (int c = grp; c < nc; c += kPivGroups) {
        int64_t p = pp[c];
        if (p == wpos) p = P;
        else if (p == P) p = wpos;
        if (sub == 0) pp[c] = p;
        if (p <= P) continue;
        double* col = W + (size_t)c * sP;
        if (tau != 0.0) {
          double w0 = 0.0, w1 = 0.0;
          for (int i = j + sub, q = 0; i < s; i += 4, ++q) {
            if (q & 1) w1 = fma(vv[i], col[i], w1);
            else w0 = fma(vv[i], col[i], w0);
          }
          double wsum = w0 + w1;
          wsum += __shfl_xor_sync(gmask, wsum, 1);
          wsum += __shfl_xor_sync(gmask, wsum, 2);
          const double wt = wsum * tau;
          for (int i = j + sub; i < s; i += 4) col[i] = fma(-vv[i], wt, col[i]);
        }
        __syncwarp(gmask);
        const double rj = col[j];
        double rr = r[c] - rj * rj;
        if (rr < 1e-8 * r0[c] || rr < 0.0) {
          double t = 0.0;
          for (int i = j + 1 + sub; i < s; i += 4) t = fma(col[i], col[i], t);
          t += __shfl_xor_sync(gmask, t, 1);
          t += __shfl_xor_sync(gmask, t, 2);
          rr = t > 0.0 ? t : 0.0;
        }
        if (sub == 0) r[c] = rr;
        cand_push(cd, rr, p);
      }
    } else {
      for (int c = grp; c < nc; c += kPivGroups) {
        int64_t p = pp[c];
        if (p == wpos) p = P;
        else if (p == P) p = wpos;
        if (sub == 0) pp[c] = p;
        if (p <= P) continue;
        double* col = W + (size_t)c * sP;
        // rows j.. of the column in registers (s <= 128: <= 32 per thread): one L2
        // round trip per column for the load, none for row j or the guard recompute
        constexpr int kSQ = 32;
        double x[kSQ];
#pragma unroll
        for (int q = 0; q < kSQ; ++q) {
          const int i = j + sub + 4 * q;
          x[q] = i < s ? col[i] : 0.0;
        }
        if (tau != 0.0) {
          double w0 = 0.0, w1 = 0.0;
#pragma unroll
          for (int q = 0; q < kSQ; ++q) {
            const int i = j + sub + 4 * q;
            if (i < s) {
              if (q & 1) w1 = fma(vv[i], x[q], w1);
              else w0 = fma(vv[i], x[q], w0);
            }
          }
          double wsum = w0 + w1;
          wsum += __shfl_xor_sync(gmask, wsum, 1);
          wsum += __shfl_xor_sync(gmask, wsum, 2);
          const double wt = wsum * tau;
#pragma unroll
          for (int q = 0; q < kSQ; ++q) {
            const int i = j + sub + 4 * q;
            if (i < s) {
              x[q] = fma(-vv[i], wt, x[q]);
              col[i] = x[q];
            }
          }
        }
        const double rj = __shfl_sync(gmask, x[0], lane & ~3);   // row j: sub 0, q 0
        double rr = r[c] - rj * rj;
        if (rr < 1e-8 * r0[c] || rr < 0.0) {
          double t = 0.0;
#pragma unroll
          for (int q = 0; q < kSQ; ++q) {
            const int i = j + sub + 4 * q;
            if (i > j && i < s) t = fma(x[q], x[q], t);
          }
          t += __shfl_xor_sync(gmask, t, 1);
          t += __shfl_xor_sync(gmask, t, 2);
          rr = t > 0.0 ? t : 0.0;
        }
        if (sub == 0) r[c] = rr;
        cand_push(cd, rr, p);
      }
    }
    if (a.gap) {
      cd = warp_top2(cd);
    } else {
      warp_best(cd.r1, cd.p1);
      cd.r2 = -1.0;
      cd.p2 = -1;
    }
    if (lane == 0) wc[warp] = cd;
    __syncthreads();
    PPROF(5)
  }
#undef PPROF
  if (a.prof && tid == 0)
    for (int i = 0; i < 6; ++i) atomicAdd((unsigned long long*)&a.prof[i], (unsigned long long)tp[i]);
  for (int c = tid; c < nc; c += kPivThreads) {
    a.pos[c0 + c] = pp[c];
    a.arr[pp[c]] = c0 + c;    // arr[pos[c]] = c: every position is owned by exactly one column
  }
}

size_t pivots_smem_bytes(int s, int cpc, bool smem_mode) {
  const int sP = pivots_stride(s);
  size_t b = (smem_mode ? (size_t)sP * cpc : 0) * sizeof(double);
  b += (size_t)cpc * (2 * sizeof(double) + sizeof(int64_t));
  b += (size_t)((s + 1) & ~1) * sizeof(double) + 8 * sizeof(Cand2) + 64;
  return b;
}

// record: [0..1] best r, [2] best position, [3] runner-up position, [4..5]
// runner-up r, [6..7] pad, then rows 0..s-1 of the candidate column (2 words each)
int pivots_recw(int s) { return (8 + 2 * s + 15) / 16 * 16; }

int pivots_stride(int s) {
  int sP = s;
  while (sP % 16 != 4) ++sP;
  return sP;
}

int pivots_rq(int s, int cpc, bool smem_mode) {
  if (!smem_mode && s <= 48) return -2;
  if (s > 128) return -1;
  if (!smem_mode || cpc > kPivGroups) return 0;
  return s <= 32 ? 8 : s <= 64 ? 16 : s <= 96 ? 24 : 32;
}

void* pivots_kernel_ptr(bool smem_mode, int rq, int s) {
  if (s > 256) return smem_mode ? (void*)pivots_kernel<true, -1, 16> : (void*)pivots_kernel<false, -1, 16>;
  if (s > 128) return smem_mode ? (void*)pivots_kernel<true, -1, 8> : (void*)pivots_kernel<false, -1, 8>;
  if (!smem_mode) return rq == -2 ? (void*)pivots_kernel<false, -2, 4> : (void*)pivots_kernel<false, 0, 4>;
  switch (rq) {
    case 8: return (void*)pivots_kernel<true, 8, 4>;
    case 16: return (void*)pivots_kernel<true, 16, 4>;
    case 24: return (void*)pivots_kernel<true, 24, 4>;
    case 32: return (void*)pivots_kernel<true, 32, 4>;
    default: return (void*)pivots_kernel<true, 0, 4>;
  }
}

cudaError_t launch_pivots(cudaStream_t st, const PivotArgs& a, bool smem_mode, size_t smem) {
  PivotArgs args = a;
  args.sP = pivots_stride(a.s);
  static long long* prof = nullptr;
  if (getenv("FFB_PIV_PROF") && !prof) cudaMallocManaged(&prof, 8 * sizeof(long long));
  if (prof) {
    for (int i = 0; i < 8; ++i) prof[i] = 0;
    args.prof = prof;
  }
  void* kargs[] = {&args};
  if (a.s > 512) return cudaErrorInvalidValue;
  const int rq = pivots_rq(a.s, a.cpc, smem_mode);
  void* kern = pivots_kernel_ptr(smem_mode, rq, a.s);
  // one per-device opt-in mask per kernel instance of pivots_kernel_ptr
  static std::atomic<unsigned long long> attr_done[11];
  const int ki = a.s > 256 ? 6 + smem_mode : a.s > 128 ? 8 + smem_mode
               : !smem_mode ? (rq == -2 ? 10 : 0) : rq == 8 ? 1 : rq == 16 ? 2 : rq == 24 ? 3 : rq == 32 ? 4 : 5;
  ensure_smem_optin(kern, 210 * 1024, attr_done[ki]);
  cudaError_t e = cudaLaunchCooperativeKernel(kern, dim3(a.G),
                                              dim3(kPivThreads), kargs, smem, st);
  if (prof && e == cudaSuccess) {
    cudaStreamSynchronize(st);
    const double d = (double)a.G * a.bb;
    fprintf(stderr,
            "[piv prof] G=%d bb=%d s=%d cpc=%d cycles/step: publish %.0f wait %.0f pick %.0f refl %.0f "
            "sync %.0f apply %.0f\n",
            a.G, a.bb, a.s, a.cpc, prof[0] / d, prof[1] / d, prof[2] / d, prof[3] / d, prof[4] / d,
            prof[5] / d);
  }
  return e;
}

// ------------------------------------------------------- gathers / copies

// element (i, c) of src at src[i * rs + c * cs] (column-major: rs = 1, cs = ld)
__global__ void gather_cols_kernel(const double* __restrict__ src, int64_t rs, int64_t cs, int64_t rows,
                                   const int64_t* __restrict__ idx, int64_t ncols,
                                   double* __restrict__ dst, int64_t ld_dst) {
  const int64_t j = blockIdx.y;
  const int64_t c = idx[j];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i + j * ld_dst] = src[i * rs + c * cs];
}

cudaError_t launch_gather_cols_strided(cudaStream_t st, const double* src, int64_t rs, int64_t cs,
                                       int64_t rows, const int64_t* idx, int64_t ncols, double* dst,
                                       int64_t ld_dst) {
  if (rows <= 0 || ncols <= 0) return cudaSuccess;
  unsigned gx = nblk(rows, 256);
  if (gx > 64) gx = 64;
  gather_cols_kernel<<<dim3(gx, (unsigned)ncols), 256, 0, st>>>(src, rs, cs, rows, idx, ncols, dst,
                                                                 ld_dst);
  FFB_LAUNCH_CHECK();
}

cudaError_t launch_gather_cols(cudaStream_t st, const double* src, int64_t ld_src, int64_t rows,
                               const int64_t* idx, int64_t ncols, double* dst, int64_t ld_dst) {
  return launch_gather_cols_strided(st, src, 1, ld_src, rows, idx, ncols, dst, ld_dst);
}

// dst[idx[c], j] = src[c, j]
__global__ void scatter_rows_kernel(const double* __restrict__ src, int64_t ld_src, int64_t nrows,
                                    int64_t ncols, const int64_t* __restrict__ idx,
                                    double* __restrict__ dst, int64_t ld_dst) {
  const int64_t total = nrows * ncols;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = t % nrows, j = t / nrows;
    dst[idx[c] + j * ld_dst] = src[c + j * ld_src];
  }
}

cudaError_t launch_scatter_rows(cudaStream_t st, const double* src, int64_t ld_src, int64_t nrows,
                                int64_t ncols, const int64_t* idx, double* dst, int64_t ld_dst) {
  const int64_t total = nrows * ncols;
  if (total <= 0) return cudaSuccess;
  unsigned g = nblk(total, 256);
  if (g > 4096) g = 4096;
  scatter_rows_kernel<<<g, 256, 0, st>>>(src, ld_src, nrows, ncols, idx, dst, ld_dst);
  FFB_LAUNCH_CHECK();
}

__global__ void copy2d_kernel(const double* __restrict__ src, int64_t ld_src, int64_t rows,
                              int64_t cols, double* __restrict__ dst, int64_t ld_dst) {
  const int64_t total = rows * cols;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t % rows, j = t / rows;
    dst[i + j * ld_dst] = src[i + j * ld_src];
  }
}

cudaError_t launch_copy_rows(cudaStream_t st, const double* src, int64_t ld_src, int64_t rows,
                             int64_t cols, double* dst, int64_t ld_dst) {
  const int64_t total = rows * cols;
  if (total <= 0) return cudaSuccess;
  unsigned g = nblk(total, 256);
  if (g > 8192) g = 8192;
  copy2d_kernel<<<g, 256, 0, st>>>(src, ld_src, rows, cols, dst, ld_dst);
  FFB_LAUNCH_CHECK();
}

// rows x cols block of a ROW-major source (src[i * ld_src + j]) into column-major dst
// (reads coalesced along j, one row per warp-stride)
__global__ void copy2d_rm_kernel(const double* __restrict__ src, int64_t ld_src, int64_t rows,
                                 int64_t cols, double* __restrict__ dst, int64_t ld_dst) {
  const int64_t total = rows * cols;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = t % cols, i = t / cols;
    dst[i + j * ld_dst] = src[i * ld_src + j];
  }
}

cudaError_t launch_copy_rows_rm(cudaStream_t st, const double* src, int64_t ld_src, int64_t rows,
                                int64_t cols, double* dst, int64_t ld_dst) {
  const int64_t total = rows * cols;
  if (total <= 0) return cudaSuccess;
  unsigned g = nblk(total, 256);
  if (g > 8192) g = 8192;
  copy2d_rm_kernel<<<g, 256, 0, st>>>(src, ld_src, rows, cols, dst, ld_dst);
  FFB_LAUNCH_CHECK();
}

// Byte copy on the SMs (8-byte words + tail).  Used for every small transfer and
// device-to-device copy on the engine's stream, with pinned host buffers
// addressed directly (UVA), so no copy-engine queue -- where another stream's
// large H2D/D2H may be in flight -- sits on a factorization's critical path.
__global__ void copy_bytes_kernel(const unsigned char* __restrict__ src, unsigned char* __restrict__ dst,
                                  size_t bytes) {
  const size_t nw = bytes >> 3;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const size_t t0 = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if ((((uintptr_t)src | (uintptr_t)dst) & 7) == 0) {
    const unsigned long long* s8 = reinterpret_cast<const unsigned long long*>(src);
    unsigned long long* d8 = reinterpret_cast<unsigned long long*>(dst);
    for (size_t t = t0; t < nw; t += stride) d8[t] = s8[t];
    for (size_t t = (nw << 3) + t0; t < bytes; t += stride) dst[t] = src[t];
  } else {
    for (size_t t = t0; t < bytes; t += stride) dst[t] = src[t];
  }
}

cudaError_t launch_copy_bytes(cudaStream_t st, const void* src, void* dst, size_t bytes) {
  if (bytes == 0) return cudaSuccess;
  size_t g = ((bytes >> 3) + 255) / 256;
  if (g < 1) g = 1;
  if (g > 2048) g = 2048;
  copy_bytes_kernel<<<(unsigned)g, 256, 0, st>>>(static_cast<const unsigned char*>(src),
                                                 static_cast<unsigned char*>(dst), bytes);
  FFB_LAUNCH_CHECK();
}

__global__ void fill_kernel(double* p, size_t count, double v) {
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < count;
       t += (size_t)gridDim.x * blockDim.x)
    p[t] = v;
}

cudaError_t launch_fill(cudaStream_t st, double* p, size_t count, double v) {
  if (!count) return cudaSuccess;
  unsigned g = nblk((int64_t)count, 256);
  if (g > 8192) g = 8192;
  fill_kernel<<<g, 256, 0, st>>>(p, count, v);
  FFB_LAUNCH_CHECK();
}

__global__ void add_identity_kernel(double* X, int64_t ld, int64_t nd, double scale) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nd;
       i += (int64_t)gridDim.x * blockDim.x)
    X[i + i * ld] += scale;
}

cudaError_t launch_add_identity(cudaStream_t st, double* X, int64_t ld, int64_t rows,
                                int64_t cols, double scale) {
  const int64_t nd = rows < cols ? rows : cols;
  if (nd <= 0) return cudaSuccess;
  add_identity_kernel<<<nblk(nd, 256) > 256 ? 256 : nblk(nd, 256), 256, 0, st>>>(X, ld, nd, scale);
  FFB_LAUNCH_CHECK();
}

__global__ void add_top_kernel(double* X, int64_t ldx, const double* Y, int64_t ldy, int64_t rows,
                               int64_t cols) {
  const int64_t total = rows * cols;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t % rows, j = t / rows;
    X[i + j * ldx] += Y[i + j * ldy];
  }
}

cudaError_t launch_add_top(cudaStream_t st, double* X, int64_t ldx, const double* Y, int64_t ldy,
                           int64_t rows, int64_t cols) {
  const int64_t total = rows * cols;
  if (total <= 0) return cudaSuccess;
  unsigned g = nblk(total, 256);
  if (g > 4096) g = 4096;
  add_top_kernel<<<g, 256, 0, st>>>(X, ldx, Y, ldy, rows, cols);
  FFB_LAUNCH_CHECK();
}

__global__ void finite_check_kernel(const double* x, size_t count, uint32_t* status) {
  bool bad = false;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < count;
       t += (size_t)gridDim.x * blockDim.x)
    bad |= !isfinite(x[t]);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(status, kStNonFinite);
}

cudaError_t launch_finite_check(cudaStream_t st, const double* x, size_t count, uint32_t* status) {
  if (!count) return cudaSuccess;
  unsigned g = nblk((int64_t)count, 256);
  if (g > 1184) g = 1184;
  finite_check_kernel<<<g, 256, 0, st>>>(x, count, status);
  FFB_LAUNCH_CHECK();
}

// ------------------------------------- panel reconstruction (K4 / K12)
//
// A Householder panel (rows x w, w <= 64) is factored as shifted CholeskyQR3
// (Gram -> Cholesky -> X R^-1, three passes; first pass shifted by
// 11(Mw + w(w+1)) u tr(G), Fukaya et al. 2020) followed by the Householder
// reconstruction of Ballard et al.: LU without pivoting of Q_top*D - I where
// the sign D_c is chosen so that every pivot is <= -1.  This reproduces the
// reflectors of LAPACK-style Householder QR with the reference's sign rule
// alpha = -sign(x0)||x|| (ffsrqr/qr.py:21-43, _kernels_numpy.py:84-109):
// Q - E = Y (-T Y1^T) is exactly that LU, with pivot -tau_c in [-2,-1].  A
// pivot of exactly 0 (|z| == 1) is the reference's identity-reflector branch.

constexpr int kMaxW = 64;
constexpr int kSLD = kMaxW + 1;

// Gram G (w x w, reduced), optional shift, Cholesky (upper R, R^T R = G),
// R^-1, and Racc <- R * Racc (Racc := R when `first`).  One CTA, 256 threads.
__global__ void __launch_bounds__(256) cholinv_kernel(const double* __restrict__ Gin, int w,
                                                      int64_t rows_m, int shift, int first,
                                                      double* Racc, double* Rinv,
                                                      uint32_t* status) {
  extern __shared__ __align__(16) double dsm[];
  double* G = dsm;
  double* R = G + kMaxW * kSLD;
  double* X = R + kMaxW * kSLD;
  __shared__ double red[8];
  __shared__ int bad;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int ww = w * w;
  if (tid == 0) bad = 0;
  for (int t = tid; t < ww; t += nt) {
    const int i = t % w, j = t / w;
    G[i * kSLD + j] = Gin[t];
    R[i * kSLD + j] = 0.0;
    X[i * kSLD + j] = 0.0;
  }
  __syncthreads();
  double tr = 0.0;
  for (int i = tid; i < w; i += nt) tr += G[i * kSLD + i];
  tr = block_sum(tr, red);
  if (tr == 0.0) {
    // all-zero panel: R = I, R^-1 = I, Racc := 0 (first) / unchanged.  signlu
    // then emits identity reflectors (reference's tail == 0 branch).
    for (int t = tid; t < ww; t += nt) {
      const int i = t % w, j = t / w;
      Rinv[i + j * w] = (i == j) ? 1.0 : 0.0;
      if (first) Racc[i + j * w] = 0.0;
    }
    return;
  }
  if (shift) {
    const double sh = 11.0 * ((double)rows_m * w + (double)w * (w + 1)) * 1.1102230246251565e-16 * tr;
    for (int i = tid; i < w; i += nt) G[i * kSLD + i] += sh;
    __syncthreads();
  }
  // right-looking Cholesky on the upper triangle: 2 barriers per column; thread
  // (tx = column q, ty = row phase) layout, no integer division in the loop
  {
    const int tx = tid & 63, ty = tid >> 6, nty = nt >> 6;
    for (int j = 0; j < w; ++j) {
      double d = G[j * kSLD + j];
      if (!(d > 0.0) || !isfinite(d)) {
        if (tid == 0) bad = 1;
        d = d > 0.0 ? d : 1e-300;
      }
      const double rjj = sqrt(d);
      if (ty == 0 && tx >= j && tx < w) R[j * kSLD + tx] = (tx == j) ? rjj : G[j * kSLD + tx] / rjj;
      __syncthreads();
      if (tx > j && tx < w) {
        const double rq = R[j * kSLD + tx];
        for (int k = j + 1 + ty; k <= tx; k += nty) G[k * kSLD + tx] -= R[j * kSLD + k] * rq;
      }
      __syncthreads();
    }
  }
  // X = R^-1 by rows from the bottom; 4 lanes per column share each dot.
  {
    const int c = tid >> 2, sub = tid & 3;
    for (int i = w - 1; i >= 0; --i) {
      double acc = 0.0;
      if (c < w && c >= i)
        for (int k = i + 1 + sub; k <= c; k += 4) acc = fma(R[i * kSLD + k], X[k * kSLD + c], acc);
      acc += __shfl_xor_sync(0xffffffffu, acc, 1);
      acc += __shfl_xor_sync(0xffffffffu, acc, 2);
      if (c < w && c >= i && sub == 0) X[i * kSLD + c] = ((i == c ? 1.0 : 0.0) - acc) / R[i * kSLD + i];
      __syncthreads();
    }
  }
  // new Racc = R * Racc (upper x upper), staged in G
  for (int t = tid; t < ww; t += nt) {
    const int i = t % w, j = t / w;
    Rinv[i + j * w] = X[i * kSLD + j];
    double acc = 0.0;
    if (first) {
      acc = R[i * kSLD + j];
    } else if (i <= j) {
      for (int k = i; k <= j; ++k) acc = fma(R[i * kSLD + k], Racc[k + j * w], acc);
    }
    G[i * kSLD + j] = acc;
  }
  __syncthreads();
  for (int t = tid; t < ww; t += nt) {
    const int i = t % w, j = t / w;
    Racc[i + j * w] = G[i * kSLD + j];
  }
  if (tid == 0 && bad) atomicOr(status, kStCholFail);
}

cudaError_t launch_cholinv(cudaStream_t st, const double* G, int w, int64_t rows_m, bool shift,
                           bool first, double* Racc, double* Rinv, uint32_t* status) {
  constexpr int kSm = 3 * kMaxW * kSLD * sizeof(double);
  static std::atomic<unsigned long long> init{0};
  ensure_smem_optin((const void*)cholinv_kernel, kSm, init);
  cholinv_kernel<<<1, 256, kSm, st>>>(G, w, rows_m, shift ? 1 : 0, first ? 1 : 0, Racc, Rinv,
                                       status);
  FFB_LAUNCH_CHECK();
}

// LU of Q_top*D - I with per-column sign choice; emits L (into Y's top w rows),
// T = -U L^{-T}, R = D*Racc (upper), D, and Ut = D * U^{-1} (zero-pivot columns
// zeroed) so that the lower reflector rows are Y2 = Q_bottom * Ut.  One CTA.
__global__ void __launch_bounds__(256) signlu_kernel(const double* __restrict__ Qtop, int64_t ldq,
                                                     int w, const double* __restrict__ Racc,
                                                     double* Y, int64_t ldy, double* T,
                                                     int64_t ldt, double* Rout, int64_t ldr,
                                                     double* Ut, double* Dout) {
  extern __shared__ __align__(16) double dsm[];
  double* q = dsm;
  double* L = q + kMaxW * kSLD;
  double* U = L + kMaxW * kSLD;
  double* Ui = U + kMaxW * kSLD;      // D * U^{-1}
  double* Ts = Ui + kMaxW * kSLD;     // T
  __shared__ double Dd[kMaxW];
  const int tid = threadIdx.x, nt = blockDim.x;
  bool zero_panel = true;
  for (int i = 0; i < w; ++i) zero_panel &= (Racc[i + i * w] == 0.0);
  if (zero_panel) {
    for (int t = tid; t < w * w; t += nt) {
      const int i = t % w, j = t / w;
      Y[i + j * ldy] = (i == j) ? 1.0 : 0.0;
      T[i + j * ldt] = 0.0;
      Rout[i + j * ldr] = 0.0;
      Ut[i + j * w] = 0.0;
    }
    for (int i = tid; i < w; i += nt) Dout[i] = 1.0;
    return;
  }
  for (int t = tid; t < w * w; t += nt) {
    const int i = t % w, j = t / w;
    q[i * kSLD + j] = Qtop[i + j * ldq];
    L[i * kSLD + j] = (i == j) ? 1.0 : 0.0;
    U[i * kSLD + j] = 0.0;
  }
  __syncthreads();
  for (int c = 0; c < w; ++c) {
    // every thread derives the same sign from q[c][c] (no extra barrier)
    const double z = q[c * kSLD + c];
    double d;
    if (fabs(z) == 1.0) d = z > 0.0 ? 1.0 : -1.0;    // identity reflector (tail == 0)
    else d = z > 0.0 ? -1.0 : 1.0;                   // pivot -(1+|z|) = -tau
    const double ucc = d * z - 1.0;
    if (tid == 0) {
      Dd[c] = d;
      U[c * kSLD + c] = ucc;
    }
    for (int i = c + 1 + tid; i < w; i += nt) L[i * kSLD + c] = ucc != 0.0 ? d * q[i * kSLD + c] / ucc : 0.0;
    for (int k = tid; k < c; k += nt) U[k * kSLD + c] = d * q[k * kSLD + c];
    __syncthreads();
    {
      const int tx = tid & 63, ty = tid >> 6, nty = nt >> 6;
      if (tx > c && tx < w) {
        const double qc = q[c * kSLD + tx];
        for (int i = c + 1 + ty; i < w; i += nty) q[i * kSLD + tx] -= L[i * kSLD + c] * qc;
      }
    }
    __syncthreads();
  }
  // Column-sequential solves, all rows in parallel (4 lanes per row):
  //   Ui row i: y U = e_i  -> y_c = (delta_ic - sum_{k<c} y_k U[k][c]) / U[c][c]
  //   T  row i: t L^T = -U[i,:] -> t_c = -U[i][c] - sum_{k<c} t_k L[c][k]
  {
    const int i = tid >> 2, sub = tid & 3;
    for (int c = 0; c < w; ++c) {
      double a0 = 0.0, a1 = 0.0;
      if (i < w)
        for (int k = sub; k < c; k += 4) {
          a0 = fma(Ui[i * kSLD + k], U[k * kSLD + c], a0);
          a1 = fma(Ts[i * kSLD + k], L[c * kSLD + k], a1);
        }
      a0 += __shfl_xor_sync(0xffffffffu, a0, 1);
      a0 += __shfl_xor_sync(0xffffffffu, a0, 2);
      a1 += __shfl_xor_sync(0xffffffffu, a1, 1);
      a1 += __shfl_xor_sync(0xffffffffu, a1, 2);
      if (i < w && sub == 0) {
        const double ucc = U[c * kSLD + c];
        Ui[i * kSLD + c] = ucc != 0.0 ? ((i == c ? 1.0 : 0.0) - a0) / ucc : 0.0;
        Ts[i * kSLD + c] = -U[i * kSLD + c] - a1;
      }
      __syncthreads();
    }
  }
  for (int t = tid; t < w * w; t += nt) {
    const int i = t % w, j = t / w;
    Y[i + j * ldy] = L[i * kSLD + j];
    T[i + j * ldt] = Ts[i * kSLD + j];
    Ut[i + j * w] = Dd[i] * Ui[i * kSLD + j];
    Rout[i + j * ldr] = (i <= j) ? Dd[i] * Racc[i + j * w] : 0.0;
  }
  for (int i = tid; i < w; i += nt) Dout[i] = Dd[i];
}

cudaError_t launch_signlu(cudaStream_t st, const double* Qtop, int64_t ldq, int w,
                          const double* Racc, double* Y, int64_t ldy, double* T, int64_t ldt,
                          double* R, int64_t ldr, double* Ut, double* D) {
  constexpr int kSm = 5 * kMaxW * kSLD * sizeof(double);
  static std::atomic<unsigned long long> init{0};
  ensure_smem_optin((const void*)signlu_kernel, kSm, init);
  signlu_kernel<<<1, 256, kSm, st>>>(Qtop, ldq, w, Racc, Y, ldy, T, ldt, R, ldr, Ut, D);
  FFB_LAUNCH_CHECK();
}

// ------------------------------------------------------ TRQRCP helpers

// R rows j0..j0+bb: entries at arrangement positions < j0 are exact zeros and the
// block's own columns take the panel's upper-triangular R (alpha on the
// diagonal, ffsrqr/sketch.py:137-139).
__global__ void fix_rrows_kernel(double* R, int64_t ldr, int64_t j0, int bb,
                                 const int64_t* __restrict__ arr, const double* __restrict__ Rb,
                                 int64_t ldrb) {
  const int64_t e = j0 + bb;
  const int64_t total = (int64_t)bb * e;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(t % bb);
    const int64_t p = t / bb;
    const int64_t col = arr[p];
    double v = 0.0;
    if (p >= j0 && p - j0 >= i) v = Rb[i + (p - j0) * ldrb];
    R[(j0 + i) + col * ldr] = v;
  }
}

cudaError_t launch_fix_rrows(cudaStream_t st, double* R, int64_t ldr, int64_t j0, int bb,
                             const int64_t* arr, const double* Rb, int64_t ldrb) {
  const int64_t total = (int64_t)bb * (j0 + bb);
  fix_rrows_kernel<<<nblk(total, 256) > 1024 ? 1024 : nblk(total, 256), 256, 0, st>>>(
      R, ldr, j0, bb, arr, Rb, ldrb);
  FFB_LAUNCH_CHECK();
}

// Rinv = Rb^{-1} for an upper-triangular w x w Rb (w <= 64), so that the sketch
// update Z = B_piv Rb^{-1} runs as one DMMA GEMM.  Exact zero pivots (only an
// all-zero panel produces them) give zero rows and raise kStZeroPivot; the
// reference would fall back to lstsq there (ffsrqr/sketch.py:75-83).
__global__ void __launch_bounds__(256) triinv_upper_kernel(const double* __restrict__ Rb,
                                                           int64_t ldrb, int w, double* Rinv,
                                                           int64_t ldo, uint32_t* status) {
  using namespace tile64;
  extern __shared__ __align__(16) double dsm[];
  double* U = dsm;                 // 64 x kTL
  double* X = U + 64 * kTL;        // 64 x kTL
  double* S = X + 64 * kTL;        // 1024 scratch
  __shared__ int zp;
  const int tid = threadIdx.x, nt = blockDim.x;
  if (tid == 0) zp = 0;
  for (int t = tid; t < 64 * 64; t += nt) {
    const int i = t >> 6, j = t & 63;
    U[i * kTL + j] = (i < w && j < w) ? Rb[i + (int64_t)j * ldrb] : 0.0;
  }
  __syncthreads();
  if (tid < w && U[tid * kTL + tid] == 0.0) zp = 1;
  inv_upper_blk(U, w, X, S);
  for (int t = tid; t < w * w; t += nt) {
    const int i = t % w, j = t / w;
    Rinv[i + j * ldo] = X[i * kTL + j];
  }
  if (tid == 0 && zp) atomicOr(status, kStZeroPivot);
}

cudaError_t launch_triinv_upper(cudaStream_t st, const double* Rb, int64_t ldrb, int w,
                                double* Rinv, int64_t ldo, uint32_t* status) {
  constexpr int kSm = (2 * 64 * tile64::kTL + 1024) * sizeof(double);
  static std::atomic<unsigned long long> init{0};
  ensure_smem_optin((const void*)triinv_upper_kernel, kSm, init);
  triinv_upper_kernel<<<1, 256, kSm, st>>>(Rb, ldrb, w, Rinv, ldo, status);
  FFB_LAUNCH_CHECK();
}

// ------------------------------------------------------------ SRQR (K7-K11)

// r[p] = ||B[:, arr[p]]||^2 / s for p >= l (sketch-based initialisation,
// ffsrqr/srqr.py:98-101); zero for p < l.
__global__ void rinit_kernel(const double* __restrict__ B, int64_t ldb, int s,
                             const int64_t* __restrict__ arr, int64_t n, int64_t l, double* r,
                             double* rinit) {
  const int lane = threadIdx.x & 31;
  const int64_t p = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (p >= n) return;
  double v = 0.0;
  if (p >= l) {
    const double* b = B + arr[p] * ldb;
    double acc = 0.0;
    for (int i = lane; i < s; i += 32) acc = fma(b[i], b[i], acc);
    v = warp_sum(acc) / (double)s;
  }
  if (lane == 0) {
    r[p] = v;
    rinit[p] = v;
  }
}

cudaError_t launch_rinit(cudaStream_t st, const double* B, int64_t ldb, int s, const int64_t* arr,
                         int64_t n, int64_t l, double* r, double* rinit) {
  rinit_kernel<<<nblk(n, 8), 256, 0, st>>>(B, ldb, s, arr, n, l, r, rinit);
  FFB_LAUNCH_CHECK();
}

__global__ void anorm_kernel(const double* __restrict__ colsq, int64_t n, SrqrScalars* sc) {
  __shared__ double red[32];
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) acc += colsq[i];
  acc = block_sum(acc, red);
  if (threadIdx.x == 0) {
    sc->anorm = sqrt(acc);
    sc->status = isfinite(acc) ? 0u : kStNonFinite;
    sc->need_swap = 0;
    sc->alpha = 0.0;
    sc->g2 = 0.0;
  }
}

cudaError_t launch_anorm(cudaStream_t st, const double* colsq, int64_t n, SrqrScalars* sc) {
  anorm_kernel<<<1, 1024, 0, st>>>(colsq, n, sc);
  FFB_LAUNCH_CHECK();
}

// piv = l + argmax r[l:] (ties -> lowest position); swap into position l
// (ffsrqr/srqr.py:121-123, swap_cols 109-115).
__global__ void __launch_bounds__(1024) ext_pick_kernel(int64_t l, int64_t n, int64_t* arr,
                                                        int64_t* pos, double* r, double* rinit,
                                                        SrqrScalars* sc) {
  __shared__ double red_v[32];
  __shared__ int64_t red_i[32];
  ArgMax best{-1.0, -1};
  for (int64_t p = l + threadIdx.x; p < n; p += blockDim.x) best = argmax_better(best, ArgMax{r[p], p});
  best = block_argmax(best, red_v, red_i);
  if (threadIdx.x == 0) {
    const int64_t q = best.i < 0 ? l : best.i;
    sc->piv = q;
    if (q != l) {
      const int64_t a = arr[l], b = arr[q];
      arr[l] = b;
      arr[q] = a;
      pos[b] = l;
      pos[a] = q;
      double t = r[l];
      r[l] = r[q];
      r[q] = t;
      t = rinit[l];
      rinit[l] = rinit[q];
      rinit[q] = t;
    }
  }
}

cudaError_t launch_ext_pick(cudaStream_t st, int64_t l, int64_t n, int64_t* arr, int64_t* pos,
                            double* r, double* rinit, SrqrScalars* sc) {
  ext_pick_kernel<<<1, 1024, 0, st>>>(l, n, arr, pos, r, rinit, sc);
  FFB_LAUNCH_CHECK();
}

// u = A[:, c] - Q1 R[:l, c]   (c = arr[l])
__global__ void ext_u_kernel(const double* __restrict__ A, int64_t ars, int64_t acs, int64_t m, int64_t l,
                             const double* __restrict__ Q, int64_t ldq, const double* __restrict__ R,
                             int64_t ldr, const int64_t* __restrict__ arr, double* u) {
  extern __shared__ double rc[];
  const int64_t c = arr[l];
  for (int64_t j = threadIdx.x; j < l; j += blockDim.x) rc[j] = R[j + c * ldr];
  __syncthreads();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= m) return;
  double a0 = 0.0, a1 = 0.0;
  int64_t j = 0;
  for (; j + 1 < l; j += 2) {
    a0 = fma(Q[i + j * ldq], rc[j], a0);
    a1 = fma(Q[i + (j + 1) * ldq], rc[j + 1], a1);
  }
  if (j < l) a0 = fma(Q[i + j * ldq], rc[j], a0);
  u[i] = A[i * ars + c * acs] - (a0 + a1);
}

// ct[j] = Q[:, j]^T u  (one CTA per j, deterministic)
__global__ void ext_ct_kernel(const double* __restrict__ Q, int64_t ldq, int64_t m,
                              const double* __restrict__ u, double* ct) {
  __shared__ double red[32];
  const int64_t j = blockIdx.x;
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) acc = fma(Q[i + j * ldq], u[i], acc);
  acc = block_sum(acc, red);
  if (threadIdx.x == 0) ct[j] = acc;
}

// u -= Q1 ct  (second CGS pass, srqr.py:125); per-block partial ||u||^2
__global__ void ext_u2_kernel(const double* __restrict__ Q, int64_t ldq, int64_t m, int64_t l,
                              const double* __restrict__ ct, double* u, double* part) {
  extern __shared__ double cs[];
  __shared__ double red[32];
  for (int64_t j = threadIdx.x; j < l; j += blockDim.x) cs[j] = ct[j];
  __syncthreads();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double sq = 0.0;
  if (i < m) {
    double a0 = 0.0, a1 = 0.0;
    int64_t j = 0;
    for (; j + 1 < l; j += 2) {
      a0 = fma(Q[i + j * ldq], cs[j], a0);
      a1 = fma(Q[i + (j + 1) * ldq], cs[j + 1], a1);
    }
    if (j < l) a0 = fma(Q[i + j * ldq], cs[j], a0);
    const double v = u[i] - (a0 + a1);
    u[i] = v;
    sq = v * v;
  }
  sq = block_sum(sq, red);
  if (threadIdx.x == 0) part[blockIdx.x] = sq;
}

// alpha = ||u||; rank test alpha <= 1e-14 max(||A||_F, 1e-300) (srqr.py:127-133);
// R row l := alpha e_l (srqr.py:128,135), r[l] = alpha^2.
__global__ void ext_fin_kernel(const double* __restrict__ part, int nparts, int64_t l, int64_t n,
                               const int64_t* __restrict__ arr, double* R, int64_t ldr, double* r,
                               SrqrScalars* sc) {
  __shared__ double red[32];
  double acc = 0.0;
  for (int t = threadIdx.x; t < nparts; t += blockDim.x) acc += part[t];
  acc = block_sum(acc, red);
  double alpha = sqrt(acc);
  const double an = sc->anorm;
  if (alpha <= 1e-14 * fmax(an, 1e-300)) alpha = 0.0;
  for (int64_t c = threadIdx.x; c < n; c += blockDim.x) R[l + c * ldr] = 0.0;
  __syncthreads();
  if (threadIdx.x == 0) {
    sc->alpha = alpha;
    if (!isfinite(acc)) sc->status |= kStNonFinite;
    R[l + arr[l] * ldr] = alpha;
    if (alpha > 0.0) r[l] = alpha * alpha;
  }
}

__global__ void ext_q_kernel(const double* __restrict__ u, int64_t m, double* Ql,
                             const SrqrScalars* sc) {
  const double alpha = sc->alpha;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < m) Ql[i] = alpha > 0.0 ? u[i] / alpha : 0.0;
}

cudaError_t launch_ext_project(cudaStream_t st, const double* A, int64_t ars, int64_t acs, int64_t m, int64_t l,
                               const double* Q, int64_t ldq, const double* R, int64_t ldr,
                               const int64_t* arr, double* u, double* ct, double* part,
                               SrqrScalars* sc, double* r, double* Rfull) {
  (void)R;
  const unsigned g = nblk(m, 256);
  const size_t sh = sizeof(double) * (size_t)(l > 0 ? l : 1);
  ext_u_kernel<<<g, 256, sh, st>>>(A, ars, acs, m, l, Q, ldq, Rfull, ldr, arr, u);
  if (l > 0) {
    ext_ct_kernel<<<(unsigned)l, 256, 0, st>>>(Q, ldq, m, u, ct);
  }
  ext_u2_kernel<<<g, 256, sh, st>>>(Q, ldq, m, l, ct, u, part);
  return cudaGetLastError();
}

cudaError_t launch_ext_finish(cudaStream_t st, const double* part, int nparts, int64_t l, int64_t n,
                              const int64_t* arr, double* R, int64_t ldr, double* r,
                              SrqrScalars* sc, const double* u, int64_t m, double* Ql) {
  ext_fin_kernel<<<1, 1024, 0, st>>>(part, nparts, l, n, arr, R, ldr, r, sc);
  ext_q_kernel<<<nblk(m, 256), 256, 0, st>>>(u, m, Ql, sc);
  FFB_LAUNCH_CHECK();
}

// Extension row R[l, arr[p]] = q^T A[:, arr[p]] for p > l, downdate r and the
// guard recompute against exact_trailing_sq(i, l+1) (srqr.py:136-149).  Only
// materialised on the swap path (the row is dead when g2 <= g).
__global__ void ext_row_kernel(const double* __restrict__ A, int64_t ars, int64_t acs, int64_t m, int64_t n,
                               int64_t l, const double* __restrict__ q, double* R, int64_t ldr,
                               const int64_t* __restrict__ arr, const double* __restrict__ colsq,
                               double* r, const double* __restrict__ rinit,
                               const SrqrScalars* sc) {
  const int lane = threadIdx.x & 31;
  const int64_t p = l + 1 + (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (p >= n || !(sc->alpha > 0.0)) return;
  const int64_t col = arr[p];
  const double* a = A + col * acs;
  double acc = 0.0;
  for (int64_t i = lane; i < m; i += 32) acc = fma(q[i], a[i * ars], acc);
  acc = warp_sum(acc);
  // exact trailing norm below l+1 rows, needed only by the guard
  double rs = 0.0;
  for (int64_t i = lane; i < l; i += 32) {
    const double v = R[i + col * ldr];
    rs = fma(v, v, rs);
  }
  rs = warp_sum(rs);
  if (lane == 0) {
    R[l + col * ldr] = acc;
    double rr = r[p] - acc * acc;
    if (rr < 1e-8 * rinit[p] || rr < 0.0) rr = fmax(colsq[col] - (rs + acc * acc), 0.0);
    r[p] = rr;
  }
}

cudaError_t launch_ext_row(cudaStream_t st, const double* A, int64_t ars, int64_t acs, int64_t m, int64_t n,
                           int64_t l, const double* Q, int64_t ldq, double* R, int64_t ldr,
                           const int64_t* arr, const double* colsq, double* r,
                           const double* rinit, const SrqrScalars* sc) {
  if (n <= l + 1) return cudaSuccess;
  ext_row_kernel<<<nblk(n - l - 1, 8), 256, 0, st>>>(A, ars, acs, m, n, l, Q + l * ldq, R, ldr, arr,
                                                       colsq, r, rinit, sc);
  FFB_LAUNCH_CHECK();
}

// g2 estimate (ffsrqr/srqr.py:49-64): Z = Rtilde^{-1} Omega^T by right-looking
// back substitution; row norms; first argmax; g2 = |alpha|/sqrt(d) * max.
// Thread k owns row k of Z (its d right-hand sides live in registers).  Step i:
// the owner of row i (already final) divides by Rtilde_ii and publishes z_i;
// one barrier; every row k < i does z_k -= Rtilde_ki z_i.  Column values
// Rtilde_ki = R[k, arr[i]] are prefetched RING steps ahead with cp.async into a
// per-thread ring in shared memory (each thread only ever reads its own row, so
// the ring needs no barrier): the columns sit 2 KB apart in R, mostly out of L2
// by the time this kernel runs, and a four-deep register ring left 47 % of the
// stall samples on those loads.  Omega is d x (l+1) row-major (numpy C order).
constexpr int kG2MaxD = 16;
template <int MAXT, int RING>
__global__ void __launch_bounds__(MAXT) g2_kernel(const double* __restrict__ R, int64_t ldr,
                                                  const int64_t* __restrict__ arr, int64_t l,
                                                  const double* __restrict__ omega, int d, double g,
                                                  double* Z, SrqrScalars* sc) {
  extern __shared__ int64_t g2cols[];   // [l+1] arrangement (column of Rtilde -> R column), then the ring
  __shared__ double zb[2][kG2MaxD];
  __shared__ double red_v[32];
  __shared__ int64_t red_i[32];
  __shared__ int sing;
  const int L1 = (int)(l + 1);
  const double alpha = sc->alpha;
  const int tid = threadIdx.x, nt = blockDim.x;
  if (tid == 0) sing = 0;
  __syncthreads();
  if (!(alpha > 0.0)) {
    if (tid == 0) {
      sc->g2 = 0.0;
      sc->i_off = 0;
      sc->need_swap = 0;
    }
    return;
  }
  for (int i = tid; i < L1; i += nt) {
    const int64_t c = arr[i];
    g2cols[i] = c;
    const double dv = (i == l) ? alpha : R[i + c * ldr];
    if (dv == 0.0) sing = 1;
  }
  __syncthreads();
  if (sing) {
    if (tid == 0) {
      sc->status |= kStSingular;
      sc->need_swap = 0;
    }
    return;
  }
  const int k = tid;   // this thread's row (L1 <= 1024)
  const double dkk = k < L1 ? (k == (int)l ? alpha : R[k + g2cols[k] * ldr]) : 1.0;
  const double rdkk = 1.0 / dkk;   // the solve multiplies by the inverted diagonal
  // Rtilde_{k,col}: column l is (R[:l, arr[l]]; alpha); rows above the column only.
  // ring[slot][thread]: slot col % RING holds this row's entry of column col
  double* ring = reinterpret_cast<double*>(g2cols + ((L1 + 1) & ~1));
  auto prefetch = [&](int col) {
    const bool live = col >= 0 && k < col;
    cp_async8(ring + (size_t)((col % RING + RING) % RING) * nt + tid, live ? R + k + g2cols[col] * ldr : R, live);
    cp_async_commit();
  };
  double nrm2 = 0.0;
  for (int r0 = 0; r0 < d; r0 += kG2MaxD) {   // right-hand sides in chunks of 16
    const int dc = d - r0 < kG2MaxD ? d - r0 : kG2MaxD;
    double z[kG2MaxD];
#pragma unroll
    for (int r = 0; r < kG2MaxD; ++r)
      z[r] = (r < dc && k < L1) ? omega[(int64_t)(r0 + r) * L1 + k] : 0.0;
    for (int q = 0; q < RING; ++q) prefetch(L1 - 1 - q);
    auto step = [&](int i) {
      const int par = i & 1;
      if (k == i) {
#pragma unroll
        for (int r = 0; r < kG2MaxD; ++r)
          if (r < dc) {
            z[r] = z[r] * rdkk;
            zb[par][r] = z[r];
          }
      }
      cp_async_wait<RING - 1>();   // this thread's copy for step i has landed
      const double c = ring[(size_t)(i % RING) * nt + tid];
      __syncthreads();
      prefetch(i - RING);          // the slot now serves step i - RING
      if (k < i) {
#pragma unroll
        for (int r = 0; r < kG2MaxD; ++r)
          if (r < dc) z[r] = fma(-c, zb[par][r], z[r]);
      }
    };
    for (int i = L1 - 1; i >= 0; --i) step(i);
    cp_async_wait<0>();
#pragma unroll
    for (int r = 0; r < kG2MaxD; ++r)
      if (r < dc) nrm2 = fma(z[r], z[r], nrm2);
    __syncthreads();
  }
  ArgMax best{-1.0, -1};
  if (k < L1) best = ArgMax{sqrt(nrm2), (int64_t)k};
  best = block_argmax(best, red_v, red_i);
  if (tid == 0) {
    const double g2 = fabs(alpha) / sqrt((double)d) * best.v;
    sc->g2 = g2;
    sc->i_off = best.i;
    sc->need_swap = g2 > g ? 1u : 0u;
  }
  (void)Z;
}

cudaError_t launch_g2(cudaStream_t st, const double* R, int64_t ldr, const int64_t* arr, int64_t l,
                      const double* omega, int d, double g, double* Z, SrqrScalars* sc) {
  if (l + 1 > 1024) return cudaErrorInvalidValue;
  const int threads = (int)((l + 1 + 31) / 32 * 32);
  const int ring = threads <= 512 ? 32 : 16;
  const size_t smem = sizeof(int64_t) * (size_t)((l + 2) & ~1) + sizeof(double) * (size_t)ring * threads;
  static std::atomic<unsigned long long> attr_done[2];
  if (threads <= 512) {
    ensure_smem_optin((const void*)g2_kernel<512, 32>, 200 * 1024, attr_done[0]);
    g2_kernel<512, 32><<<1, threads, smem, st>>>(R, ldr, arr, l, omega, d, g, Z, sc);
  } else {
    ensure_smem_optin((const void*)g2_kernel<1024, 16>, 200 * 1024, attr_done[1]);
    g2_kernel<1024, 16><<<1, threads, smem, st>>>(R, ldr, arr, l, omega, d, g, Z, sc);
  }
  FFB_LAUNCH_CHECK();
}

// ---- g2 for l + 1 > 1024 (srqr.py:49-64): Z = Rtilde^{-1} Omega^T by blocked
// back substitution on an explicit Rtilde — diagonal blocks of <= 1024 rows
// solved one thread per row (as g2_kernel), the rows above updated by one
// engine GEMM per block — then row norms and the first-max argmax.

// Rt (L1 x L1, upper, from launch_r_arranged): diagonal (l, l) <- alpha;
// Z (L1 x d, column-major) <- Omega^T; flag <- 1 alpha == 0, 2 singular
__global__ void g2big_prep_kernel(double* Rt, int64_t L1, const double* __restrict__ omega, int d,
                                  double* Z, const SrqrScalars* sc, uint32_t* flag) {
  const double alpha = sc->alpha;
  const int64_t tot = L1 * (int64_t)d;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / L1, k = t - r * L1;
    Z[k + r * L1] = omega[r * L1 + k];
    if (r == 0) {
      if (k == L1 - 1) Rt[k + k * L1] = alpha;
      const double dv = (k == L1 - 1) ? alpha : Rt[k + k * L1];
      if (!(alpha > 0.0)) atomicOr(flag, 1u);
      else if (dv == 0.0) atomicOr(flag, 2u);
    }
  }
}

__global__ void __launch_bounds__(1024) g2big_diag_kernel(const double* __restrict__ Rt, int64_t L1,
                                                          int64_t i0, int nbk, double* Z, int d) {
  __shared__ double zb[2][kG2MaxD];
  const int t = threadIdx.x;
  const int64_t k = i0 + t;
  const bool own = t < nbk;
  const double rd = own ? 1.0 / Rt[k + k * L1] : 1.0;
  for (int r0 = 0; r0 < d; r0 += kG2MaxD) {
    const int dc = d - r0 < kG2MaxD ? d - r0 : kG2MaxD;
    double z[kG2MaxD];
#pragma unroll
    for (int r = 0; r < kG2MaxD; ++r) z[r] = (own && r < dc) ? Z[k + (int64_t)(r0 + r) * L1] : 0.0;
    double cn = (own && t < nbk - 1) ? Rt[k + (i0 + nbk - 1) * L1] : 0.0;
    for (int i = nbk - 1; i >= 0; --i) {
      const int par = i & 1;
      if (t == i) {
#pragma unroll
        for (int r = 0; r < kG2MaxD; ++r)
          if (r < dc) {
            z[r] = z[r] * rd;
            zb[par][r] = z[r];
          }
      }
      const double c = cn;
      cn = (own && t < i - 1) ? Rt[k + (i0 + i - 1) * L1] : 0.0;   // next step's coefficient
      __syncthreads();
      if (t < i) {
#pragma unroll
        for (int r = 0; r < kG2MaxD; ++r)
          if (r < dc) z[r] = fma(-c, zb[par][r], z[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < kG2MaxD; ++r)
      if (own && r < dc) Z[k + (int64_t)(r0 + r) * L1] = z[r];
    __syncthreads();
  }
}

__global__ void __launch_bounds__(1024) g2big_finish_kernel(const double* __restrict__ Z, int64_t L1,
                                                            int d, double g, const uint32_t* flag,
                                                            SrqrScalars* sc) {
  __shared__ double red_v[32];
  __shared__ int64_t red_i[32];
  const uint32_t f = *flag;
  ArgMax best{-1.0, -1};
  for (int64_t k = threadIdx.x; k < L1; k += blockDim.x) {
    double nrm2 = 0.0;
    for (int r = 0; r < d; ++r) {
      const double z = Z[k + (int64_t)r * L1];
      nrm2 = fma(z, z, nrm2);
    }
    best = argmax_better(best, ArgMax{sqrt(nrm2), k});
  }
  best = block_argmax(best, red_v, red_i);
  if (threadIdx.x == 0) {
    if (f & 1u) {
      sc->g2 = 0.0;
      sc->i_off = 0;
      sc->need_swap = 0;
    } else if (f & 2u) {
      sc->status |= kStSingular;
      sc->need_swap = 0;
    } else {
      const double g2 = fabs(sc->alpha) / sqrt((double)d) * best.v;
      sc->g2 = g2;
      sc->i_off = best.i;
      sc->need_swap = g2 > g ? 1u : 0u;
    }
  }
}

cudaError_t launch_g2big_prep(cudaStream_t st, double* Rt, int64_t L1, const double* omega, int d,
                              double* Z, const SrqrScalars* sc, uint32_t* flag) {
  cudaError_t e = cudaMemsetAsync(flag, 0, sizeof(uint32_t), st);
  if (e != cudaSuccess) return e;
  unsigned g = nblk(L1 * (int64_t)d, 256);
  if (g > 4096) g = 4096;
  g2big_prep_kernel<<<g, 256, 0, st>>>(Rt, L1, omega, d, Z, sc, flag);
  FFB_LAUNCH_CHECK();
}

cudaError_t launch_g2big_diag(cudaStream_t st, const double* Rt, int64_t L1, int64_t i0, int nbk,
                              double* Z, int d) {
  g2big_diag_kernel<<<1, (nbk + 31) / 32 * 32, 0, st>>>(Rt, L1, i0, nbk, Z, d);
  FFB_LAUNCH_CHECK();
}

cudaError_t launch_g2big_finish(cudaStream_t st, const double* Z, int64_t L1, int d, double g,
                                const uint32_t* flag, SrqrScalars* sc) {
  g2big_finish_kernel<<<1, 1024, 0, st>>>(Z, L1, d, g, flag, sc);
  FFB_LAUNCH_CHECK();
}

// _pack (srqr.py:213-235): trail_sq = max(colsq - ||R[:l, c]||^2, 0) over
// positions >= l; r22 = sqrt(max); g1 = r22/alpha; tau bounds.
__global__ void pack_part_kernel(const double* __restrict__ R, int64_t ldr,
                                 const int64_t* __restrict__ arr, const double* __restrict__ colsq,
                                 int64_t l, int64_t n, double* part) {
  __shared__ double wmax[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double mx = 0.0;
  for (int64_t p = l + (int64_t)blockIdx.x * nw + wid; p < n; p += (int64_t)gridDim.x * nw) {
    const int64_t col = arr[p];
    const double* rc = R + col * ldr;
    double acc = 0.0;
    for (int64_t i = lane; i < l; i += 32) acc = fma(rc[i], rc[i], acc);
    acc = warp_sum(acc);
    mx = fmax(mx, fmax(colsq[col] - acc, 0.0));
  }
  if (lane == 0) wmax[wid] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < nw; ++w) t = fmax(t, wmax[w]);
    part[blockIdx.x] = t;
  }
}

__global__ void pack_fin_kernel(const double* __restrict__ part, int nparts, int64_t l, int64_t n,
                                SrqrScalars* sc) {
  if (threadIdx.x != 0) return;
  double t = 0.0;
  for (int q = 0; q < nparts; ++q) t = fmax(t, part[q]);
  const double r22 = (n > l) ? sqrt(t) : 0.0;
  const double alpha = sc->alpha;
  const double g1 = alpha > 0.0 ? r22 / alpha : 0.0;
  const double g2 = alpha > 0.0 ? sc->g2 : 0.0;
  sc->r22 = r22;
  sc->g1 = g1;
  sc->tau = g1 * g2 * sqrt((double)(l + 1) * (double)(n - l));
  sc->tau_hat = g1 * g2 * sqrt((double)l * (double)(n - l));
}

cudaError_t launch_pack(cudaStream_t st, const double* R, int64_t ldr, const int64_t* arr,
                        const double* colsq, int64_t l, int64_t n, double* part, int64_t swaps,
                        SrqrScalars* sc) {
  (void)swaps;
  const int nparts = 148;
  pack_part_kernel<<<nparts, 256, 0, st>>>(R, ldr, arr, colsq, l, n, part);
  pack_fin_kernel<<<1, 32, 0, st>>>(part, nparts, l, n, sc);
  FFB_LAUNCH_CHECK();
}

// rotate_out (srqr.py:152-164): cyclic left shift of positions i_off..l, then
// the Givens chase of qr.py:182-209 (rotations computed sequentially from the
// diagonal columns, identical arithmetic to row-wise application), applied to
// every column of R and to the columns of Q (qr.py:212-219).
__global__ void rot_compute_kernel(double* R, int64_t ldr, int64_t l, int64_t* arr, int64_t* pos,
                                   double* r, double* rinit, const SrqrScalars* sc, double* rot,
                                   double* scratch) {
  if (threadIdx.x != 0) return;
  const int64_t i_off = sc->i_off;
  if (i_off < l) {
    const int64_t a0 = arr[i_off];
    const double r0 = r[i_off], q0 = rinit[i_off];
    for (int64_t p = i_off; p < l; ++p) {
      arr[p] = arr[p + 1];
      r[p] = r[p + 1];
      rinit[p] = rinit[p + 1];
      pos[arr[p]] = p;
    }
    arr[l] = a0;
    r[l] = r0;
    rinit[l] = q0;
    pos[a0] = l;
  }
  // rotations: for i = i_off..l-1 on rows (i, i+1), from column arr[i]
  for (int64_t i = i_off; i < l; ++i) {
    const int64_t col = arr[i];
    // column entries rows i_off..i+1 after rotations i_off..i-1
    double* x = scratch;
    for (int64_t k = i_off; k <= i + 1; ++k) x[k - i_off] = R[k + col * ldr];
    for (int64_t k = i_off; k < i; ++k) {
      const double c = rot[3 * k], s = rot[3 * k + 1];
      if (rot[3 * k + 2] != 0.0) continue;
      const double up = c * x[k - i_off] + s * x[k + 1 - i_off];
      const double lo = -s * x[k - i_off] + c * x[k + 1 - i_off];
      x[k - i_off] = up;
      x[k + 1 - i_off] = lo;
    }
    const double a = x[i - i_off], b = x[i + 1 - i_off];
    if (b == 0.0) {
      rot[3 * i] = 1.0;
      rot[3 * i + 1] = 0.0;
      rot[3 * i + 2] = 1.0;  // skipped
    } else {
      const double h = hypot(a, b);
      rot[3 * i] = a / h;
      rot[3 * i + 1] = b / h;
      rot[3 * i + 2] = 0.0;
    }
  }
}

__global__ void rot_apply_R_kernel(double* R, int64_t ldr, int64_t n, int64_t l,
                                   const int64_t* __restrict__ arr, const double* __restrict__ rot,
                                   const SrqrScalars* sc) {
  const int64_t i_off = sc->i_off;
  for (int64_t col = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; col < n;
       col += (int64_t)gridDim.x * blockDim.x) {
    double* rc = R + col * ldr;
    for (int64_t i = i_off; i < l; ++i) {
      if (rot[3 * i + 2] != 0.0) continue;
      const double c = rot[3 * i], s = rot[3 * i + 1];
      const double a = rc[i], b = rc[i + 1];
      rc[i] = c * a + s * b;
      rc[i + 1] = -s * a + c * b;
    }
  }
}

__global__ void rot_zero_kernel(double* R, int64_t ldr, int64_t l, const int64_t* __restrict__ arr,
                                const double* __restrict__ rot, const SrqrScalars* sc) {
  const int64_t i_off = sc->i_off;
  for (int64_t i = i_off + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < l;
       i += (int64_t)gridDim.x * blockDim.x)
    if (rot[3 * i + 2] == 0.0) R[(i + 1) + arr[i] * ldr] = 0.0;
}

__global__ void rot_apply_Q_kernel(double* Q, int64_t ldq, int64_t m, int64_t l,
                                   const double* __restrict__ rot, const SrqrScalars* sc) {
  const int64_t i_off = sc->i_off;
  for (int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; row < m;
       row += (int64_t)gridDim.x * blockDim.x) {
    for (int64_t i = i_off; i < l; ++i) {
      if (rot[3 * i + 2] != 0.0) continue;
      const double c = rot[3 * i], s = rot[3 * i + 1];
      const double q0 = Q[row + i * ldq], q1 = Q[row + (i + 1) * ldq];
      Q[row + i * ldq] = c * q0 + s * q1;
      Q[row + (i + 1) * ldq] = -s * q0 + c * q1;
    }
  }
}

cudaError_t launch_rotate_out(cudaStream_t st, double* R, int64_t ldr, double* Q, int64_t ldq,
                              int64_t m, int64_t n, int64_t l, int64_t* arr, int64_t* pos,
                              double* r, double* rinit, const SrqrScalars* sc, double* rot) {
  double* scratch = rot + 3 * (l + 1);
  rot_compute_kernel<<<1, 32, 0, st>>>(R, ldr, l, arr, pos, r, rinit, sc, rot, scratch);
  rot_apply_R_kernel<<<nblk(n, 256) > 1184 ? 1184 : nblk(n, 256), 256, 0, st>>>(R, ldr, n, l, arr,
                                                                                  rot, sc);
  rot_zero_kernel<<<nblk(l + 1, 256), 256, 0, st>>>(R, ldr, l, arr, rot, sc);
  rot_apply_Q_kernel<<<nblk(m, 256) > 1184 ? 1184 : nblk(m, 256), 256, 0, st>>>(Q, ldq, m, l, rot,
                                                                                  sc);
  FFB_LAUNCH_CHECK();
}

// revert_extension (srqr.py:166-171)
__global__ void revert_kernel(const double* __restrict__ R, int64_t ldr,
                              const int64_t* __restrict__ arr, int64_t l, int64_t n, double* r) {
  for (int64_t p = l + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    const double v = R[l + arr[p] * ldr];
    if (p == l) r[p] = v * v;
    else r[p] += v * v;
  }
}

cudaError_t launch_revert(cudaStream_t st, const double* R, int64_t ldr, const int64_t* arr,
                          int64_t l, int64_t n, double* r) {
  revert_kernel<<<nblk(n - l, 256) > 1184 ? 1184 : nblk(n - l, 256), 256, 0, st>>>(R, ldr, arr, l,
                                                                                    n, r);
  FFB_LAUNCH_CHECK();
}

// ------------------------------------------------------------- outputs

// out[i, c] = R[i, arr[c]] for i < rows, zero below the diagonal for i < tri_rows
__global__ void r_arranged_kernel(const double* __restrict__ R, int64_t ldr,
                                  const int64_t* __restrict__ arr, int64_t rows, int64_t n,
                                  double* out, int64_t ldo, int64_t tri_rows) {
  const int64_t total = rows * n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t % rows, c = t / rows;
    out[i + c * ldo] = (i > c && i < tri_rows) ? 0.0 : R[i + arr[c] * ldr];
  }
}

cudaError_t launch_r_arranged(cudaStream_t st, const double* R, int64_t ldr, const int64_t* arr,
                              int64_t rows, int64_t n, double* out, int64_t ldo,
                              int64_t tri_rows) {
  const int64_t total = rows * n;
  if (total <= 0) return cudaSuccess;
  unsigned g = nblk(total, 256);
  if (g > 8192) g = 8192;
  r_arranged_kernel<<<g, 256, 0, st>>>(R, ldr, arr, rows, n, out, ldo, tri_rows);
  FFB_LAUNCH_CHECK();
}

// X = (R arranged, upper trapezoidal)^T : X[c, i] = R[i, arr[c]] for i <= c
__global__ void build_rt_kernel(const double* __restrict__ R, int64_t ldr,
                                const int64_t* __restrict__ arr, int64_t l, int64_t n, double* X,
                                int64_t ldx) {
  const int64_t total = l * n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = t % n, i = t / n;
    X[c + i * ldx] = (i <= c) ? R[i + arr[c] * ldr] : 0.0;
  }
}

cudaError_t launch_build_rt(cudaStream_t st, const double* R, int64_t ldr, const int64_t* arr,
                            int64_t l, int64_t n, double* X, int64_t ldx) {
  const int64_t total = l * n;
  unsigned g = nblk(total, 256);
  if (g > 8192) g = 8192;
  build_rt_kernel<<<g, 256, 0, st>>>(R, ldr, arr, l, n, X, ldx);
  FFB_LAUNCH_CHECK();
}

__global__ void diag_kernel(const double* R, int64_t ldr, int64_t nd, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nd;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = R[i + i * ldr];
}

cudaError_t launch_diag(cudaStream_t st, const double* R, int64_t ldr, int64_t nd, double* out) {
  diag_kernel<<<nblk(nd, 256), 256, 0, st>>>(R, ldr, nd, out);
  FFB_LAUNCH_CHECK();
}

}  // namespace ffb
