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

#include <algorithm>
#include <stdio.h>
#include <stdlib.h>

#include "ffb_common.cuh"
#include "ffb_jacobi.cuh"

#include <cooperative_groups.h>
namespace cg = cooperative_groups;

namespace ffb {

namespace {

constexpr int kJThreads = 256;
constexpr int kMW = 36;   // smem row stride (doubles): 16-byte rows, conflict-free DMMA fragments

FFB_DEV uint32_t ld_acq(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
FFB_DEV void st_rel(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

// Grid barrier on one monotone counter (bar[0], zero at launch): the k-th
// barrier completes when the counter reaches k * nblocks.  Arrival is a
// fire-and-forget red.release, the wait polls with ld.acquire — one L2 round
// trip on the critical path (ffb_panel.cu has the same barrier).  `passed`
// counts the barriers this thread has been through.
FFB_DEV void grid_barrier(uint32_t* bar, uint32_t nblocks, uint32_t& passed) {
  ++passed;
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(bar) : "memory");
    const uint32_t target = passed * nblocks;
    while (ld_acq(bar) < target) {
    }
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
FFB_DEV bool rotation(const double* G, int p, int q, double tol2, double& c, double& s,
                      double& c2, double& den, bool kLeanRotation) {
  c = 1.0;
  s = 0.0;
  c2 = 0.0;
  den = 1.0;
  // padding slots hold zero columns: aa * bb = 0 fails the threshold test below
  const double aa = G[p * kMW + p], bb = G[q * kMW + q], cc = G[p * kMW + q];
  c2 = cc * cc;
  den = aa * bb;
  if (!(c2 > tol2 * den)) return false;
  if (kLeanRotation) {
    // tan(theta) = sign(d) g / (|d| + h), d = bb - aa, g = 2 cc, h = hypot(d, g):
    //   c = sqrt((h + |d|) / 2h),  s = sign(d) g / (2 h c)
    // in fp32 from power-of-two-normalised (d, g) (two MUFU.RSQ), then (c, s)
    // renormalised in fp64 by the second-order series of 1/sqrt(c^2 + s^2)
    const double d = bb - aa, g = cc + cc;
    const int ex = (__double2hiint(fabs(d) + fabs(g)) >> 20) & 0x7ff;
    const double scale = __hiloint2double((2046 - ex) << 20, 0);
    const float df = (float)(d * scale), gf = (float)(g * scale);
    const float rh = rsqrtf(fmaf(df, df, gf * gf));
    const float h2 = fmaf(0.5f * fabsf(df), rh, 0.5f);
    const float rc = rsqrtf(h2);
    const float cf = h2 * rc;
    const float sf = copysignf(0.5f * rh * rc, df) * gf;
    const double cd = (double)cf, sd = (double)sf;
    const double e = fma(sd, sd, fma(cd, cd, -1.0));   // c^2 in [0.5, 1]: c^2 - 1 is exact
    const double r = fma(e, fma(e, 0.375, -0.5), 1.0);
    c = cd * r;
    s = sd * r;
    return true;
  }
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

// CLUSTER: the P CTAs form one thread-block cluster and rounds are separated by
// the hardware cluster barrier (release/acquire at cluster scope covers the
// global M, V); otherwise a cooperative grid barrier.
template <bool CLUSTER>
FFB_DEV void round_barrier(uint32_t* bar, uint32_t P, uint32_t& passed) {
  if (CLUSTER) {
    __syncthreads();
    cg::this_cluster().sync();
  } else {
    grid_barrier(bar, P, passed);
  }
}

// Layout: M and V live in global memory ROW-major with padded shape lpad x ncp
// (ncp = nb * kBS, zero padding), so a slot block of one row is 128 contiguous
// bytes: staging is 16-byte cp.async, results go back as 16-byte stores, and no
// bounds checks are needed anywhere.  Shared tiles are R x 32 row-major (kMW).

// stage rows [r0, r0 + R) of the two slot blocks (pa | pb) of X into S
FFB_DEV void stage_rows_async(double* S, const double* X, int64_t ld, int pa, int pb, int r0,
                              int R) {
  for (int idx = threadIdx.x; idx < R * 16; idx += blockDim.x) {
    const int rr = idx >> 4, ch = idx & 15;
    const int blk = ch < 8 ? pa : pb;
    const double* src = X + (int64_t)(r0 + rr) * ld + blk * kBS + (ch & 7) * 2;
    cp_async16(S + rr * kMW + (ch < 8 ? 0 : kBS) + (ch & 7) * 2, src, true);
  }
}

// X rows [r0, r0 + R) of blocks (pa | pb) <- S J (S: R x 32 in smem), 16-byte
// stores.  Warp w owns row tiles w, w + 8, .. (<= kMaxRT) x all 4 column tiles:
// up to 28 independent DMMA accumulator chains per warp.
FFB_DEV void apply_rows(const double* S, int R, const double* Js, double* X, int64_t ld, int pa,
                        int pb, int r0) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int fr = lane >> 2, fk = lane & 3;
  const int nrt = R >> 3;
  constexpr int kMaxRT = 7;
  int col[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int c = 8 * j + 2 * fk;
    col[j] = (c < kBS ? pa : pb) * kBS + (c & (kBS - 1));
  }
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
      for (int j = 0; j < 4; ++j) bf[j] = Js[(k0 + fk) * kMW + 8 * j + fr];
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
      const int64_t row = r0 + rt * 8 + fr;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        double2 v;
        v.x = acc[i][j][0];
        v.y = acc[i][j][1];
        *reinterpret_cast<double2*>(X + row * ld + col[j]) = v;
      }
    }
  }
}

// V accumulation replayed concurrently with the Jacobi rounds (fused launch):
// V = prod over rounds of the block-diagonal rotations J recorded per visit.
// Every ROW of V evolves independently (row <- row J on the pair's 32 columns),
// so replay CTA v owns rows [8v, 8v + 8) in shared memory and applies each round
// as soon as the Jacobi CTAs publish it (a.progress, release/acquire), warp w
// taking pair slots w, w + 8, .. (disjoint columns) with DMMA 8 x 32 x 32.  The
// replay runs on otherwise idle SMs, off the Jacobi critical path.
FFB_DEV void v_apply_pair(double* vr, int ldv, const double* J, int pa, int pb) {
  const int lane = threadIdx.x & 31, fr = lane >> 2, fk = lane & 3;
  double bf[8][4], af[8];
#pragma unroll
  for (int k = 0; k < 8; ++k)
#pragma unroll
    for (int j = 0; j < 4; ++j) bf[k][j] = J[(4 * k + fk) * 32 + 8 * j + fr];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int c = 4 * k + fk;
    af[k] = vr[fr * ldv + (c < kBS ? pa : pb) * kBS + (c & (kBS - 1))];
  }
  double acc[4][2];
#pragma unroll
  for (int j = 0; j < 4; ++j) acc[j][0] = acc[j][1] = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k)
#pragma unroll
    for (int j = 0; j < 4; ++j) dmma_884(acc[j][0], acc[j][1], af[k], bf[k][j]);
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = 8 * j + 2 * fk + h;
      vr[fr * ldv + (c < kBS ? pa : pb) * kBS + (c & (kBS - 1))] = acc[j][h];
    }
}

FFB_DEV void v_replay(const JacobiArgs& a, int vcta, double* vr) {
  __shared__ int s_go;
  const int row0 = vcta * 8;
  if (row0 >= a.lpad) return;
  const int tid = threadIdx.x, warp = tid >> 5, nw = blockDim.x >> 5;
  const int ncp = (int)a.ld, ldv = ncp + 4, nb = a.nb, P = a.P;
  for (int t = tid; t < 8 * ncp; t += blockDim.x) {
    const int rr = t / ncp, c = t - rr * ncp;
    vr[rr * ldv + c] = (row0 + rr == c && c < a.l) ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int q = 0;; ++q) {
    if (tid == 0) {
      int go;
      for (;;) {
        if (ld_acq(a.progress) > (uint32_t)q) { go = 1; break; }
        const uint32_t fin = ld_acq(a.progress + 1);
        if (fin != 0u && (uint32_t)q + 1u >= fin) { go = 0; break; }
        __nanosleep(256);
      }
      s_go = go;
    }
    __syncthreads();
    if (!s_go) break;
    const int r = q % (nb - 1);
    for (int slot = warp; slot < P; slot += nw)
      v_apply_pair(vr, ldv, a.jhist + ((size_t)q * P + slot) * 1024, rr_player(slot, r, nb),
                   rr_player(nb - 1 - slot, r, nb));
    __syncthreads();
  }
  for (int t = tid; t < 8 * ncp; t += blockDim.x) {
    const int rr = t / ncp, c = t - rr * ncp;
    a.V[(int64_t)(row0 + rr) * ncp + c] = vr[rr * ldv + c];
  }
}

template <bool CLUSTER>
__global__ void __launch_bounds__(kJThreads, 1) jacobi_kernel(JacobiArgs a) {
  extern __shared__ __align__(16) double sm[];
  const int lpad = a.lpad, nb = a.nb;
  // rows >= l of M are zero padding: stage, Gram and apply stop at l rounded up
  // to 32 (whole 4-row k-steps for each of the 8 warps)
  const int lrows = ((a.l + 31) & ~31) < lpad ? ((a.l + 31) & ~31) : lpad;
  double* Ms = sm;                        // lpad x kMW : M_W
  double* Gs = Ms + (size_t)lpad * kMW;   // 32 x kMW
  double* Js = Gs + 32 * kMW;
  double* Gs2 = Js + 32 * kMW;            // ping-pong partners of Gs / Js
  double* Js2 = Gs2 + 32 * kMW;
  double* part = Js2 + 32 * kMW;          // 4 x 32 x 33 Gram partials
  __shared__ double s_off;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  if ((int)blockIdx.x >= a.P) {   // fused launch: V replay CTAs (see v_replay)
    v_replay(a, (int)blockIdx.x - a.P, sm);
    return;
  }
  const int P = a.P;
  const double tol = a.tol;
  const double tol2 = a.tol * a.tol;
  const int64_t ld = a.ld;

  uint32_t gbn = 0;   // grid barriers passed (non-cluster launch)
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
      stage_rows_async(Ms, a.M, ld, pa, pb, 0, lrows);
      cp_async_commit();
      cp_async_wait<0>();
      __syncthreads();
      JPROF(0)
      // fresh Gram G = M_W^T M_W: warp w sums rows [w*lpad/8, (w+1)*lpad/8) for all
      // 16 output tiles (16 independent DMMA chains); fixed-order two-level reduce
      {
        // Round 0 of a sweep: the full Gram, upper tiles only (i <= j, mirrored).
        // Later rounds: only the fresh cross block M_a^T M_b (4 of the 16 8x8
        // tiles); the diagonal blocks are the rotated ones the previous owners of
        // blocks a and b left in gdiag (exact Grams of the current columns up to
        // the rounding of <= 16 two-sided updates, reset every sweep).  The
        // rotations stay exactly orthogonal whatever G they were computed from,
        // and sigma comes from fresh column norms, so only the rotation angles
        // see that rounding.
        const bool cross_only = r > 0;
        const int fr = lane >> 2, fk = lane & 3;
        double acc[4][4][2];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
        const int kr = lrows >> 3;                // rows per warp (multiple of 4)
        if (cross_only) {
          for (int k0 = warp * kr; k0 < (warp + 1) * kr; k0 += 4) {
            double f[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) f[i] = Ms[(k0 + fk) * kMW + 8 * i + fr];
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
              for (int j = 2; j < 4; ++j) dmma_884(acc[i][j][0], acc[i][j][1], f[i], f[j]);
          }
        } else {
          for (int k0 = warp * kr; k0 < (warp + 1) * kr; k0 += 4) {
            double f[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) f[i] = Ms[(k0 + fk) * kMW + 8 * i + fr];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
              for (int j = i; j < 4; ++j) dmma_884(acc[i][j][0], acc[i][j][1], f[i], f[j]);
          }
        }
        double* pw = part + (warp & 3) * 32 * 33;
        if (warp >= 4) {
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = i; j < 4; ++j)
#pragma unroll
              for (int h = 0; h < 2; ++h) pw[(8 * i + fr) * 33 + 8 * j + 2 * fk + h] = acc[i][j][h];
        }
        __syncthreads();
        if (warp < 4) {
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = i; j < 4; ++j)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                double& d = pw[(8 * i + fr) * 33 + 8 * j + 2 * fk + h];
                d = acc[i][j][h] + d;
              }
        }
        __syncthreads();
        const double* da = a.gdiag + (size_t)pa * kBS * kBS;
        const double* db = a.gdiag + (size_t)pb * kBS * kBS;
        for (int t = tid; t < 32 * 32; t += nt) {
          const int rr = t >> 5, c = t & 31;
          const int ru = rr < c ? rr : c, cu = rr < c ? c : rr;   // upper-triangle source
          const int o = ru * 33 + cu;
          double g;
          if (cross_only && (rr < kBS) == (c < kBS))
            g = rr < kBS ? da[rr * kBS + c] : db[(rr - kBS) * kBS + (c - kBS)];
          else
            g = (part[o] + part[32 * 33 + o]) + (part[2 * 32 * 33 + o] + part[3 * 32 * 33 + o]);
          Gs[rr * kMW + c] = g;
          Js[rr * kMW + c] = rr == c ? 1.0 : 0.0;
        }
        __syncthreads();
      }
      JPROF(1)
      // A visit whose pairs all pass the threshold test leaves M_W unchanged
      // (J = I): skip the rotation chain and the write-back.  This is the
      // converged tail of the last sweeps; the test is rotation()'s.
      __shared__ int s_active;
      if (tid == 0) s_active = 0;
      __syncthreads();
      {
        bool act = false;
        for (int t = tid; t < 32 * 32; t += nt) {
          const int p = t >> 5, q = t & 31;
          if (p >= q || (r != 0 && !(p < kBS && q >= kBS))) continue;
          const double gpq = Gs[p * kMW + q];
          act |= gpq * gpq > tol2 * (Gs[p * kMW + p] * Gs[q * kMW + q]);
        }
        if (__any_sync(0xffffffffu, act) && lane == 0) s_active = 1;
      }
      __syncthreads();
      const bool active = s_active != 0;
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
      auto step = [&](int pa2, int qa2, int pb2, int qb2) {
        const int ra = pa2 * kMW, rq = qa2 * kMW;
        const double g00 = Gc[ra + pb2], g01 = Gc[ra + qb2];
        const double g10 = Gc[rq + pb2], g11 = Gc[rq + qb2];
        const double j00 = Jc[ra + pb2], j01 = Jc[ra + qb2];
        const double j10 = Jc[rq + pb2], j11 = Jc[rq + qb2];
        double cb, sb, c2b, denb;
        const bool rot = rotation(Gc, pb2, qb2, tol2, cb, sb, c2b, denb, a.lean != 0);
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
        Gn[ra + pb2] = ca * h00 - sa * h10;
        Gn[ra + qb2] = ca * h01 - sa * h11;
        Gn[rq + pb2] = sa * h00 + ca * h10;
        Gn[rq + qb2] = sa * h01 + ca * h11;
        // J rows (pa, qa) x columns (pb, qb): J <- J R_b (column rotation only)
        Jn[ra + pb2] = cb * j00 - sb * j01;
        Jn[ra + qb2] = sb * j00 + cb * j01;
        Jn[rq + pb2] = cb * j10 - sb * j11;
        Jn[rq + qb2] = sb * j10 + cb * j11;
        __syncthreads();
        const double* tg = Gc;
        Gc = Gn;
        Gn = const_cast<double*>(tg);
        const double* tj = Jc;
        Jc = Jn;
        Jn = const_cast<double*>(tj);
      };
      for (int t = 0; active && t < n_within; ++t) {
        int pa2, qa2, pb2, qb2;
        inner_pair(t, ba, n_within, pa2, qa2);
        inner_pair(t, bb2, n_within, pb2, qb2);
        step(pa2, qa2, pb2, qb2);
      }
      // cross pairs (k, kBS + (k + t) % kBS): index math without branches
      for (int t = 0; active && t < n_cross; ++t) {
        const int tt = t & (kBS - 1);
        step(ba, kBS + ((ba + tt) & (kBS - 1)), bb2, kBS + ((bb2 + tt) & (kBS - 1)));
      }
      double off = offn > 0.0 ? sqrt(offn / offd) : 0.0;
      // the rotated diagonal blocks travel with their columns to the next owners
      {
        double* da = a.gdiag + (size_t)pa * kBS * kBS;
        double* db = a.gdiag + (size_t)pb * kBS * kBS;
        for (int t = tid; t < 2 * kBS * kBS; t += nt) {
          const int blk = t / (kBS * kBS), e = t - blk * kBS * kBS, rr = e / kBS, c = e - rr * kBS;
          const int o = blk * kBS;
          (blk ? db : da)[e] = Gc[(o + rr) * kMW + o + c];
        }
      }
      JPROF(2)
      if (active) apply_rows(Ms, lrows, Jc, a.M, ld, pa, pb, 0);
      // record this visit's J for the deferred V accumulation (jacobi_v_kernel)
      {
        double* jh = a.jhist + (((size_t)sweep * (nb - 1) + r) * P + blockIdx.x) * 1024;
        for (int t = tid; t < 1024; t += nt) jh[t] = Jc[(t >> 5) * kMW + (t & 31)];
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
      round_barrier<CLUSTER>(a.bar, P, gbn);
      // publish progress to the V replay CTAs: J of every finished round is visible
      if (a.fused && tid == 0 && blockIdx.x == 0) {
        __threadfence();
        st_rel(a.progress, (uint32_t)(sweep * (nb - 1) + r + 1));
      }
      JPROF(5)
    }
    const double om = *((volatile double*)(a.offmax + sweep));
    if (tid == 0 && blockIdx.x == 0) *a.sweeps = sweep + 1;
    // converged when no pair exceeded tol; a sweep whose largest |cos| was below
    // 1e-8 leaves only second-order (~1e-16) off-diagonal mass behind it
    // (quadratic convergence), so the confirming sweep is skipped
    if (!(om > tol) || om < 1e-8 || sweep + 1 == a.max_sweeps) {
      if (a.fused && tid == 0 && blockIdx.x == 0) st_rel(a.progress + 1, (uint32_t)((sweep + 1) * (nb - 1) + 1));
      break;
    }
  }
  if (a.prof && tid == 0 && blockIdx.x == 0)
    for (int i = 0; i < 6; ++i) a.prof[i] = tp[i];
#undef JPROF
}

// ---------------------------------------------------------------------------
// General geometry (l > 512: more block pairs than one cluster holds, columns
// taller than shared memory).  The same block one-sided Jacobi as
// jacobi_kernel, with three changes:
//   * `grid` cooperative CTAs take the P pair slots of a round round-robin
//     (slot = blockIdx.x, + grid, ...), so P may exceed the co-resident CTAs;
//   * a pair's 32 columns are streamed through shared memory in chunks of
//     kRC rows: the Gram accumulates over the chunks, the rotation chain runs
//     on the reduced 32 x 32 Gram, and the apply re-stages each chunk (M stays
//     L2-resident up to l ~ 2000: 32 MB);
//   * V is rotated in place with the same J (row-major like M) instead of
//     replaying a recorded J history (which would grow as sweeps x l^2 x 32).
constexpr int kRC = 256;   // rows per staged chunk

FFB_DEV void gram_chunk(const double* Ms, int R, bool cross_only, double (&acc)[4][4][2]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, fr = lane >> 2, fk = lane & 3;
  const int kr = R >> 3;   // rows per warp (multiple of 4)
  for (int k0 = warp * kr; k0 < (warp + 1) * kr; k0 += 4) {
    double f[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) f[i] = Ms[(k0 + fk) * kMW + 8 * i + fr];
    if (cross_only) {
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 2; j < 4; ++j) dmma_884(acc[i][j][0], acc[i][j][1], f[i], f[j]);
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = i; j < 4; ++j) dmma_884(acc[i][j][0], acc[i][j][1], f[i], f[j]);
    }
  }
}

__global__ void __launch_bounds__(kJThreads, 1) jacobi_general_kernel(JacobiArgs a) {
  extern __shared__ __align__(16) double sm[];
  const int lpad = a.lpad, nb = a.nb, P = a.P;
  const int lrows = ((a.l + 31) & ~31) < lpad ? ((a.l + 31) & ~31) : lpad;
  const bool resident = lrows <= kRC;   // one chunk: staged once, reused by the apply
  uint32_t gbn = 0;                     // grid barriers passed
  double* Ms = sm;                      // kRC x kMW
  double* Gs = Ms + (size_t)kRC * kMW;
  double* Js = Gs + 32 * kMW;
  double* Gs2 = Js + 32 * kMW;
  double* Js2 = Gs2 + 32 * kMW;
  double* part = Js2 + 32 * kMW;        // 4 x 32 x 33 Gram partials
  __shared__ double s_off;
  __shared__ int s_active;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const double tol = a.tol, tol2 = a.tol * a.tol;
  const int64_t ld = a.ld;
  for (int sweep = 0; sweep < a.max_sweeps; ++sweep) {
    if (tid == 0) s_off = 0.0;
    for (int r = 0; r < nb - 1; ++r) {
      for (int slot = blockIdx.x; slot < P; slot += gridDim.x) {
        const int pa = rr_player(slot, r, nb), pb = rr_player(nb - 1 - slot, r, nb);
        const bool cross_only = r > 0;
        // ---- Gram over the row chunks
        const int fr = lane >> 2, fk = lane & 3;
        double acc[4][4][2];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
        for (int c0 = 0; c0 < lrows; c0 += kRC) {
          const int R = lrows - c0 < kRC ? lrows - c0 : kRC;
          __syncthreads();   // previous chunk's readers are done with Ms
          stage_rows_async(Ms, a.M, ld, pa, pb, c0, R);
          cp_async_commit();
          cp_async_wait<0>();
          __syncthreads();
          gram_chunk(Ms, R, cross_only, acc);
        }
        double* pw = part + (warp & 3) * 32 * 33;
        if (warp >= 4) {
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = i; j < 4; ++j)
#pragma unroll
              for (int h = 0; h < 2; ++h) pw[(8 * i + fr) * 33 + 8 * j + 2 * fk + h] = acc[i][j][h];
        }
        __syncthreads();
        if (warp < 4) {
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = i; j < 4; ++j)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                double& d = pw[(8 * i + fr) * 33 + 8 * j + 2 * fk + h];
                d = acc[i][j][h] + d;
              }
        }
        __syncthreads();
        {
          const double* da = a.gdiag + (size_t)pa * kBS * kBS;
          const double* db = a.gdiag + (size_t)pb * kBS * kBS;
          for (int t = tid; t < 32 * 32; t += nt) {
            const int rr = t >> 5, c = t & 31;
            const int ru = rr < c ? rr : c, cu = rr < c ? c : rr;
            const int o = ru * 33 + cu;
            double g;
            if (cross_only && (rr < kBS) == (c < kBS))
              g = rr < kBS ? da[rr * kBS + c] : db[(rr - kBS) * kBS + (c - kBS)];
            else
              g = (part[o] + part[32 * 33 + o]) + (part[2 * 32 * 33 + o] + part[3 * 32 * 33 + o]);
            Gs[rr * kMW + c] = g;
            Js[rr * kMW + c] = rr == c ? 1.0 : 0.0;
          }
        }
        if (tid == 0) s_active = 0;
        __syncthreads();
        {
          bool act = false;
          for (int t = tid; t < 32 * 32; t += nt) {
            const int p = t >> 5, q = t & 31;
            if (p >= q || (r != 0 && !(p < kBS && q >= kBS))) continue;
            const double gpq = Gs[p * kMW + q];
            act |= gpq * gpq > tol2 * (Gs[p * kMW + p] * Gs[q * kMW + q]);
          }
          if (__any_sync(0xffffffffu, act) && lane == 0) s_active = 1;
        }
        __syncthreads();
        const bool active = s_active != 0;
        // ---- rotation chain (as jacobi_kernel)
        double offn = 0.0, offd = 1.0;
        const int n_within = (r == 0) ? kBS - 1 : 0;
        const int n_cross = a.inner * kBS;
        const int ba = tid >> 4, bb2 = tid & 15;
        const double* Gc = Gs;
        const double* Jc = Js;
        double* Gn = Gs2;
        double* Jn = Js2;
        auto step = [&](int pa2, int qa2, int pb2, int qb2) {
          const int ra = pa2 * kMW, rq = qa2 * kMW;
          const double g00 = Gc[ra + pb2], g01 = Gc[ra + qb2];
          const double g10 = Gc[rq + pb2], g11 = Gc[rq + qb2];
          const double j00 = Jc[ra + pb2], j01 = Jc[ra + qb2];
          const double j10 = Jc[rq + pb2], j11 = Jc[rq + qb2];
          double cb, sb, c2b, denb;
          const bool rot = rotation(Gc, pb2, qb2, tol2, cb, sb, c2b, denb, a.lean != 0);
          const double ca = __shfl_sync(0xffffffffu, cb, ba);
          const double sa = __shfl_sync(0xffffffffu, sb, ba);
          if (rot && ba == bb2 && c2b * offd > offn * denb) {
            offn = c2b;
            offd = denb;
          }
          const double h00 = cb * g00 - sb * g01, h01 = sb * g00 + cb * g01;
          const double h10 = cb * g10 - sb * g11, h11 = sb * g10 + cb * g11;
          Gn[ra + pb2] = ca * h00 - sa * h10;
          Gn[ra + qb2] = ca * h01 - sa * h11;
          Gn[rq + pb2] = sa * h00 + ca * h10;
          Gn[rq + qb2] = sa * h01 + ca * h11;
          Jn[ra + pb2] = cb * j00 - sb * j01;
          Jn[ra + qb2] = sb * j00 + cb * j01;
          Jn[rq + pb2] = cb * j10 - sb * j11;
          Jn[rq + qb2] = sb * j10 + cb * j11;
          __syncthreads();
          const double* tg = Gc;
          Gc = Gn;
          Gn = const_cast<double*>(tg);
          const double* tj = Jc;
          Jc = Jn;
          Jn = const_cast<double*>(tj);
        };
        for (int t = 0; active && t < n_within; ++t) {
          int pa2, qa2, pb2, qb2;
          inner_pair(t, ba, n_within, pa2, qa2);
          inner_pair(t, bb2, n_within, pb2, qb2);
          step(pa2, qa2, pb2, qb2);
        }
        for (int t = 0; active && t < n_cross; ++t) {
          const int tt = t & (kBS - 1);
          step(ba, kBS + ((ba + tt) & (kBS - 1)), bb2, kBS + ((bb2 + tt) & (kBS - 1)));
        }
        double off = offn > 0.0 ? sqrt(offn / offd) : 0.0;
        {
          double* da = a.gdiag + (size_t)pa * kBS * kBS;
          double* db = a.gdiag + (size_t)pb * kBS * kBS;
          for (int t = tid; t < 2 * kBS * kBS; t += nt) {
            const int blk = t / (kBS * kBS), e = t - blk * kBS * kBS, rr = e / kBS, c = e - rr * kBS;
            const int o = blk * kBS;
            (blk ? db : da)[e] = Gc[(o + rr) * kMW + o + c];
          }
        }
        // ---- apply J to M's and V's pair columns, chunk by chunk
        if (active) {
          for (int pass = 0; pass < 2; ++pass) {
            double* X = pass == 0 ? a.M : a.V;
            const int rows = lrows;   // V rows >= l are zero and stay zero
            for (int c0 = 0; c0 < rows; c0 += kRC) {
              const int R = rows - c0 < kRC ? rows - c0 : kRC;
              if (!(pass == 0 && resident)) {
                __syncthreads();
                stage_rows_async(Ms, X, ld, pa, pb, c0, R);
                cp_async_commit();
                cp_async_wait<0>();
              }
              __syncthreads();
              apply_rows(Ms, R, Jc, X, ld, pa, pb, c0);
            }
          }
        }
        __syncthreads();
        off = warp_max(off);
        if (lane == 0 && off > 0.0)
          atomicMax(reinterpret_cast<unsigned long long*>(&s_off),
                    (unsigned long long)__double_as_longlong(off));
      }
      __syncthreads();
      if (tid == 0 && s_off > 0.0)
        atomicMax(reinterpret_cast<unsigned long long*>(a.offmax + sweep),
                  (unsigned long long)__double_as_longlong(s_off));
      grid_barrier(a.bar, gridDim.x, gbn);
    }
    const double om = *((volatile double*)(a.offmax + sweep));
    if (tid == 0 && blockIdx.x == 0) *a.sweeps = sweep + 1;
    if (!(om > tol) || om < 1e-8 || sweep + 1 == a.max_sweeps) break;
  }
}

// V = I (row-major lpad x ncp) for the in-place V of the general kernel
__global__ void jacobi_vinit_kernel(double* Vrm, int l, int lpad, int ncp) {
  const int64_t total = (int64_t)lpad * ncp;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(idx / ncp), c = (int)(idx - (int64_t)r * ncp);
    Vrm[idx] = (r == c && r < l) ? 1.0 : 0.0;
  }
}

// Deferred V accumulation.  V = prod over (sweep, round) of the block-diagonal
// rotations J recorded by jacobi_kernel; every ROW of V evolves independently
// (row_i <- row_i J on the pair's 32 columns), so CTA g owns rows [8g, 8g + 8)
// in shared memory and replays the whole rotation history: warp w applies the
// pair slots w, w + 8, .. of each round (disjoint columns, one barrier per
// round) with DMMA (8 x 32 x 32 per pair), prefetching the next pair's J
// fragments from L2 while the current one computes.  Replaces 2 l^2 x 32 DMMA
// flops per round on the serial Jacobi critical path with a short parallel pass.
constexpr int kVRows = 8;
__global__ void __launch_bounds__(512) jacobi_v_kernel(const double* jhist, int nb, int P, int l,
                                                      int ncp, const int* sweeps, double* Vrm) {
  extern __shared__ __align__(16) double vr[];   // kVRows x (ncp + 4)
  const int ldv = ncp + 4;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int fr = lane >> 2, fk = lane & 3;
  const int row0 = blockIdx.x * kVRows;
  for (int t = tid; t < kVRows * ncp; t += blockDim.x) {
    const int rr = t / ncp, c = t - rr * ncp;
    vr[rr * ldv + c] = (row0 + rr == c && c < l) ? 1.0 : 0.0;
  }
  __syncthreads();
  const int S = sweeps[0];
  const int nrounds = S * (nb - 1);
  auto jptr = [&](int q, int slot) { return jhist + ((size_t)q * P + slot) * 1024; };
  auto load_b = [&](double (&b)[8][4], const double* J) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
      for (int j = 0; j < 4; ++j) b[k][j] = J[(4 * k + fk) * 32 + 8 * j + fr];
  };
  // one pair update: rows' 32 columns of blocks (pa | pb) <- (...) J
  auto apply = [&](const double (&b)[8][4], int pa, int pb) {
    double af[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int c = 4 * k + fk;
      af[k] = vr[fr * ldv + (c < kBS ? pa : pb) * kBS + (c & (kBS - 1))];
    }
    double acc[4][2];
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[j][0] = acc[j][1] = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
      for (int j = 0; j < 4; ++j) dmma_884(acc[j][0], acc[j][1], af[k], b[k][j]);
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = 8 * j + 2 * fk + h;
        vr[fr * ldv + (c < kBS ? pa : pb) * kBS + (c & (kBS - 1))] = acc[j][h];
      }
  };
  // one warp per pair slot (blockDim = 32 * P): every warp has exactly one item
  // per round; the next round's J fragments are in flight while this one computes
  double b0[8][4], b1[8][4];
  const int slot = warp;
  if (nrounds > 0) load_b(b0, jptr(0, slot));
  for (int q = 0; q < nrounds; q += 2) {
    {
      const int r = q % (nb - 1);
      if (q + 1 < nrounds) load_b(b1, jptr(q + 1, slot));
      apply(b0, rr_player(slot, r, nb), rr_player(nb - 1 - slot, r, nb));
      __syncthreads();
    }
    if (q + 1 < nrounds) {
      const int r = (q + 1) % (nb - 1);
      if (q + 2 < nrounds) load_b(b0, jptr(q + 2, slot));
      apply(b1, rr_player(slot, r, nb), rr_player(nb - 1 - slot, r, nb));
      __syncthreads();
    }
  }
  for (int t = tid; t < kVRows * ncp; t += blockDim.x) {
    const int rr = t / ncp, c = t - rr * ncp;
    Vrm[(int64_t)(row0 + rr) * ncp + c] = vr[rr * ldv + c];
  }
}

// Exponent e with 2^e ~ max |M| (exact power-of-two prescale) -> sweeps[1].
__global__ void jacobi_scale_kernel(const double* M, int64_t ldm, int l, int* sweeps) {
  __shared__ double red[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  double mx = 0.0;
  for (int j = warp; j < l; j += nw)
    for (int i = lane; i < l; i += 32) mx = fmax(mx, fabs(M[i + (int64_t)j * ldm]));
  mx = warp_max(mx);
  if (lane == 0) red[warp] = mx;
  __syncthreads();
  if (tid == 0) {
    mx = 0.0;
    for (int w = 0; w < nw; ++w) mx = fmax(mx, red[w]);
    sweeps[1] = (mx > 0.0 && isfinite(mx)) ? ilogb(mx) : 0;
  }
}

// Mrm = 2^-e M (row-major, lpad x ncp, zero padded)
__global__ void jacobi_layout_kernel(const double* M, int64_t ldm, int l, int lpad, int ncp,
                                     const int* sweeps, double* Mrm) {
  const double sc = ldexp(1.0, -sweeps[1]);
  const int64_t total = (int64_t)lpad * ncp;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(idx / ncp), c = (int)(idx - (int64_t)r * ncp);
    const bool in = r < l && c < l;
    Mrm[idx] = in ? sc * M[r + (int64_t)c * ldm] : 0.0;
  }
}

// sigma_j = ||M[:, j]|| (scaled; unscaled into sig), rank sort descending (ties
// by index): order, sig, scaled norms -> nrm
__global__ void jacobi_norms_kernel(const double* Mrm, int64_t ld, int l, int lpad,
                                    const int* sweeps, double* sig, int* order, double* nrm_out) {
  extern __shared__ double nrm[];
  const int tid = threadIdx.x;
  for (int j = tid; j < l; j += blockDim.x) {
    double a0 = 0.0, a1 = 0.0;
    int i = 0;
    for (; i + 1 < lpad; i += 2) {
      const double x = Mrm[(int64_t)i * ld + j], y = Mrm[(int64_t)(i + 1) * ld + j];
      a0 = fma(x, x, a0);
      a1 = fma(y, y, a1);
    }
    if (i < lpad) a0 = fma(Mrm[(int64_t)i * ld + j], Mrm[(int64_t)i * ld + j], a0);
    nrm[j] = sqrt(a0 + a1);
  }
  __syncthreads();
  const double unscale = ldexp(1.0, sweeps[1]);
  // total order even for NaN norms (non-finite input, reported afterwards by the
  // status word): NaN sorts last, so `order` is always a permutation
  auto key = [](double v) { return v == v ? v : -1.0; };
  for (int j = tid; j < l; j += blockDim.x) {
    int rank = 0;
    const double sj = key(nrm[j]);
    for (int q = 0; q < l; ++q) {
      const double kq = key(nrm[q]);
      rank += (kq > sj) || (kq == sj && q < j);
    }
    order[rank] = j;
    sig[rank] = nrm[j] * unscale;
    nrm_out[rank] = nrm[j];
  }
}

// U[:, r] = M[:, order[r]] / nrm[r] (zero column when nrm == 0), Vo[:, r] = V[:, order[r]]
__global__ void jacobi_out_kernel(const double* Mrm, const double* Vrm, int64_t ld, int l,
                                  const int* order, const double* nrm, double* U, int64_t ldu,
                                  double* Vo, int64_t ldvo) {
  const int64_t total = (int64_t)l * l;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(idx / l), i = (int)(idx - (int64_t)r * l);
    const int j = order[r];
    const double s = nrm[r];
    U[i + (int64_t)r * ldu] = s > 0.0 ? Mrm[(int64_t)i * ld + j] / s : 0.0;
    Vo[i + (int64_t)r * ldvo] = Vrm[(int64_t)i * ld + j];
  }
}

int jacobi_block_size(int l) {
  (void)l;
  return kBS;   // every inner round pairs all 32 staged slots (empty slots rotate trivially)
}

static void jacobi_geometry(int l, int& nb, int& lpad, int& ncp) {
  nb = (l + kBS - 1) / kBS;
  if (nb % 2) ++nb;
  if (nb < 2) nb = 2;
  lpad = (l + 63) & ~63;
  ncp = nb * kBS;
}

// l > 512 (more than 16 block pairs, or columns taller than one CTA's shared
// memory) runs jacobi_general_kernel; FFB_JACOBI_GENERAL=1 forces it (tests).
static bool jacobi_general(int l) {
  int nb, lpad, ncp;
  jacobi_geometry(l, nb, lpad, ncp);
  const size_t smem = sizeof(double) * ((size_t)lpad * kMW + 4 * 32 * kMW + 4 * 32 * 33);
  return nb / 2 > 16 || smem > 226 * 1024;
}

size_t jacobi_work_doubles(int l, int max_sweeps) {
  int nb, lpad, ncp;
  jacobi_geometry(l, nb, lpad, ncp);
  // Mrm, Vrm, norms, diagonal Gram blocks, and (cluster kernel only) the J
  // history (max_sweeps x rounds x pairs x 32 x 32) replayed into V
  size_t w = 2 * (size_t)lpad * ncp + (size_t)lpad + (size_t)nb * kBS * kBS;
  if (!jacobi_general(l)) w += (size_t)max_sweeps * (nb - 1) * (nb / 2) * 1024;
  return w;
}

cudaError_t launch_jacobi_scale(cudaStream_t st, const double* M, int64_t ldm, int l, int* sweeps) {
  jacobi_scale_kernel<<<1, 1024, 0, st>>>(M, ldm, l, sweeps);
  return cudaGetLastError();
}

cudaError_t launch_jacobi_svd(cudaStream_t st, int sms, const double* M, int64_t ldm, int l,
                              double* sig, double* U, int64_t ldu, double* Vo, int64_t ldvo,
                              double* work, uint32_t* bar, double* offmax, int* sweeps, int* order,
                              int max_sweeps) {
  {
    // small l: one lane group per column pair, iterate resident in one cluster's
    // shared memory (ffb_jacobi_ring.cu); FFB_JACOBI_BLOCK=1 keeps the block kernels
    if (getenv("FFB_JACOBI_BLOCK") == nullptr && getenv("FFB_JACOBI_GENERAL") == nullptr &&
        jacobi_ring_supported(l, sms))
      return launch_jacobi_ring(st, sms, M, ldm, l, sig, U, ldu, Vo, ldvo, work, offmax, sweeps, order,
                                max_sweeps);
  }
  int nb, lpad, ncp;
  jacobi_geometry(l, nb, lpad, ncp);
  const int P = nb / 2;
  double* Mrm = work;
  double* Vrm = Mrm + (size_t)lpad * ncp;
  double* nrm = Vrm + (size_t)lpad * ncp;
  double* gdiag = nrm + lpad;
  double* jhist = gdiag + (size_t)nb * kBS * kBS;
  int inner = 1;
  if (const char* e = getenv("FFB_JACOBI_INNER")) inner = atoi(e);
  if (inner < 1) inner = 1;
  static long long* prof = nullptr;
  if (getenv("FFB_JACOBI_PROF") && !prof) cudaMallocManaged(&prof, 8 * sizeof(long long));
  constexpr size_t kSmemMax = 226 * 1024;   // + static shared memory stays under the 227 KB opt-in limit
  const bool general = jacobi_general(l) || getenv("FFB_JACOBI_GENERAL") != nullptr;
  const size_t smem = general ? sizeof(double) * ((size_t)kRC * kMW + 4 * 32 * kMW + 4 * 32 * 33)
                              : sizeof(double) * ((size_t)lpad * kMW + 4 * 32 * kMW + 4 * 32 * 33);
  JacobiArgs a{Mrm, jhist, ncp, l, lpad, nb, 1e-15 * sqrt((double)l), max_sweeps, bar, offmax,
               sweeps, inner, prof, P, Vrm, bar + 2, 0, gdiag, getenv("FFB_JACOBI_ROT_OLD") ? 0 : 1};
  if (general) {
    cudaError_t e = cudaFuncSetAttribute(jacobi_general_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess) e = cudaMemsetAsync(bar, 0, 4 * sizeof(uint32_t), st);
    if (e == cudaSuccess) e = cudaMemsetAsync(offmax, 0, sizeof(double) * max_sweeps, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(gdiag, 0, sizeof(double) * (size_t)nb * kBS * kBS, st);
    if (e != cudaSuccess) return e;
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, jacobi_general_kernel, kJThreads, smem) != cudaSuccess || occ < 1)
      occ = 1;
    int grid = std::min(P, occ * sms);
    if (const char* ev = getenv("FFB_JACOBI_GRID")) grid = std::max(1, std::min(grid, atoi(ev)));   // tests: slot loop
    const int64_t total = (int64_t)lpad * ncp;
    const int g = (int)std::min<int64_t>((total + 255) / 256, 4 * sms);
    jacobi_scale_kernel<<<1, 1024, 0, st>>>(M, ldm, l, sweeps);
    jacobi_layout_kernel<<<g, 256, 0, st>>>(M, ldm, l, lpad, ncp, sweeps, Mrm);
    jacobi_vinit_kernel<<<g, 256, 0, st>>>(Vrm, l, lpad, ncp);
    void* args[] = {&a};
    e = cudaLaunchCooperativeKernel((void*)jacobi_general_kernel, dim3(grid), dim3(kJThreads), args, smem, st);
    if (e != cudaSuccess) return e;
    jacobi_norms_kernel<<<1, 1024, sizeof(double) * (size_t)l, st>>>(Mrm, ncp, l, lpad, sweeps, sig, order, nrm);
    const int go = (int)std::min<int64_t>(((int64_t)l * l + 255) / 256, 4 * sms);
    jacobi_out_kernel<<<go, 256, 0, st>>>(Mrm, Vrm, ncp, l, order, nrm, U, ldu, Vo, ldvo);
    return cudaGetLastError();
  }
  const bool cluster = P <= 16 && getenv("FFB_JACOBI_NOCLUSTER") == nullptr;
  void* kern = cluster ? (void*)jacobi_kernel<true> : (void*)jacobi_kernel<false>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemMax);
  cudaError_t e = cudaMemsetAsync(bar, 0, 4 * sizeof(uint32_t), st);
  if (e == cudaSuccess) e = cudaMemsetAsync(offmax, 0, sizeof(double) * max_sweeps, st);
  if (e != cudaSuccess) return e;
  jacobi_scale_kernel<<<1, 1024, 0, st>>>(M, ldm, l, sweeps);
  {
    const int64_t total = (int64_t)lpad * ncp;
    int g = (int)((total + 255) / 256);
    if (g > 4 * sms) g = 4 * sms;
    jacobi_layout_kernel<<<g, 256, 0, st>>>(M, ldm, l, lpad, ncp, sweeps, Mrm);
  }
  bool fused_ok = false;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  if (prof) {
    cudaEventCreate(&ev0);
    cudaEventCreate(&ev1);
    cudaEventRecord(ev0, st);
  }
  if (cluster) {
    if (P > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    // fused: cluster 0 iterates, clusters 1.. replay V concurrently (cooperative
    // launch guarantees co-residency for the progress spin-wait)
    const int vctas = lpad / kVRows;
    const int nvc = (vctas + P - 1) / P;
    const bool try_fused = getenv("FFB_JACOBI_NOFUSE") == nullptr && P * (1 + nvc) <= sms;
    for (int attempt = try_fused ? 0 : 1; attempt < 2 && !fused_ok; ++attempt) {
      a.fused = attempt == 0 ? 1 : 0;
      void* args[] = {&a};
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(a.fused ? P * (1 + nvc) : P);
      cfg.blockDim = dim3(kJThreads);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = st;
      cudaLaunchAttribute attr[2];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = P;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      attr[1].id = cudaLaunchAttributeCooperative;
      attr[1].val.cooperative = 1;
      cfg.attrs = attr;
      cfg.numAttrs = a.fused ? 2 : 1;
      e = cudaLaunchKernelExC(&cfg, kern, args);
      if (e == cudaSuccess) {
        fused_ok = a.fused != 0;
        if (!a.fused) break;
      } else {
        (void)cudaGetLastError();
        if (!a.fused) return e;
      }
    }
  } else {
    void* args[] = {&a};
    e = cudaLaunchCooperativeKernel(kern, dim3(P), dim3(kJThreads), args, smem, st);
    if (e != cudaSuccess) return e;
  }
  if (!fused_ok)
    jacobi_v_kernel<<<lpad / kVRows, 32 * P, sizeof(double) * kVRows * (ncp + 4), st>>>(
        jhist, nb, P, l, ncp, sweeps, Vrm);
  if (prof) cudaEventRecord(ev1, st);
  jacobi_norms_kernel<<<1, 1024, sizeof(double) * (size_t)l, st>>>(Mrm, ncp, l, lpad, sweeps, sig,
                                                                   order, nrm);
  {
    int g = (int)(((int64_t)l * l + 255) / 256);
    if (g > 4 * sms) g = 4 * sms;
    jacobi_out_kernel<<<g, 256, 0, st>>>(Mrm, Vrm, ncp, l, order, nrm, U, ldu, Vo, ldvo);
  }
  if (prof) {
    cudaStreamSynchronize(st);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ev0, ev1);
    fprintf(stderr, "jacobi iteration + V: %.3f ms\n", ms);
    fprintf(stderr, "jacobi phases (cycles, CTA0): stage %lld gram %lld inner %lld apply %lld off %lld barrier %lld\n",
            prof[0], prof[1], prof[2], prof[3], prof[4], prof[5]);
    double offs[64];
    int nsw = 0;
    cudaMemcpy(offs, offmax, sizeof(double) * (max_sweeps < 64 ? max_sweeps : 64), cudaMemcpyDeviceToHost);
    cudaMemcpy(&nsw, sweeps, sizeof(int), cudaMemcpyDeviceToHost);
    fprintf(stderr, "jacobi fused=%d offmax per sweep (tol %.2e):", (int)fused_ok, a.tol);
    for (int i = 0; i < nsw && i < 64; ++i) fprintf(stderr, " %.1e", offs[i]);
    fprintf(stderr, "\n");
  }
  return cudaGetLastError();
}

}  // namespace ffb
