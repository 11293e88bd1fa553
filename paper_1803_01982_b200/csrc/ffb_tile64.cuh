// Register-tiled dense kernels for w x w (w <= 64) matrices on one CTA of 256
// threads: thread t owns the 4x4 tile at rows bi = (t%16)*4, cols bj = (t/16)*4.
// Each elimination step publishes one row/column through shared memory and
// synchronises once or twice, so a 64-step factorization costs ~64 barriers and
// ~16 FMAs per thread per step instead of dependent shared-memory chains.
//
// Shared-memory matrices use a padded leading dimension kTL (65 doubles).
#pragma once
#include "ffb_common.cuh"

namespace ffb {
namespace tile64 {

constexpr int kTL = 65;

struct Tile {
  double v[4][4];
};

FFB_DEV int bi_of(int tid) { return (tid & 15) * 4; }
FFB_DEV int bj_of(int tid) { return (tid >> 4) * 4; }

FFB_DEV void load(Tile& t, const double* M, int w, bool ident_pad = false) {
  const int bi = bi_of(threadIdx.x), bj = bj_of(threadIdx.x);
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = bi + i, c = bj + j;
      t.v[i][j] = (r < w && c < w) ? M[r * kTL + c] : ((ident_pad && r == c) ? 1.0 : 0.0);
    }
}

FFB_DEV void store(const Tile& t, double* M) {
  const int bi = bi_of(threadIdx.x), bj = bj_of(threadIdx.x);
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) M[(bi + i) * kTL + bj + j] = t.v[i][j];
}

FFB_DEV void set_identity(Tile& t) {
  const int bi = bi_of(threadIdx.x), bj = bj_of(threadIdx.x);
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) t.v[i][j] = (bi + i == bj + j) ? 1.0 : 0.0;
}

// Upper Cholesky R^T R = G (G given as a tile, upper triangle used).  Writes R
// (full 64x64, zeros elsewhere) to Rs.  buf: >= 2*64 + 2 doubles of scratch.
// Non-positive pivots are clamped (returns false).
FFB_DEV bool chol_upper(Tile& g, int w, double* Rs, double* buf) {
  const int tid = threadIdx.x, bi = bi_of(tid), bj = bj_of(tid);
  double* row = buf;        // [64] current row of R
  double* dgl = buf + 64;   // [1] pivot
  bool ok = true;
  // zero R outside what we write
  for (int t = tid; t < 64 * 64; t += blockDim.x) Rs[(t >> 6) * kTL + (t & 63)] = 0.0;
  for (int j = 0; j < w; ++j) {
    // publish pivot
#pragma unroll
    for (int ii = 0; ii < 4; ++ii)
      if (j == bi + ii) {
#pragma unroll
        for (int jj = 0; jj < 4; ++jj)
          if (j == bj + jj) dgl[0] = g.v[ii][jj];
      }
    __syncthreads();
    double d = dgl[0];
    if (!(d > 0.0) || !isfinite(d)) {
      ok = false;
      d = d > 0.0 ? d : 1e-300;
    }
    const double rjj = sqrt(d), inv = 1.0 / rjj;
#pragma unroll
    for (int ii = 0; ii < 4; ++ii) {
      if (j == bi + ii) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int col = bj + c;
          if (col >= j && col < w) {
            const double r = (col == j) ? rjj : g.v[ii][c] * inv;
            row[col] = r;
            Rs[j * kTL + col] = r;
          }
        }
      }
    }
    __syncthreads();
    double rr[4], rc[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      rr[q] = (bi + q > j && bi + q < w) ? row[bi + q] : 0.0;
      rc[q] = (bj + q > j && bj + q < w) ? row[bj + q] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int c = 0; c < 4; ++c) g.v[i][c] = fma(-rr[i], rc[c], g.v[i][c]);
  }
  __syncthreads();
  return ok;
}

// X = R^{-1} for upper-triangular R in Rs (Gauss-Jordan from the bottom, one
// barrier per step, double-buffered row broadcast).  Zero pivots give zero rows
// (the reference's identity-reflector / lstsq fallbacks never divide by them).
FFB_DEV void inv_upper(const double* Rs, int w, Tile& x, double* buf) {
  const int tid = threadIdx.x, bi = bi_of(tid), bj = bj_of(tid);
  set_identity(x);
  for (int i = w - 1; i >= 0; --i) {
    double* row = buf + (i & 1) * 64;
    {
      const double d = Rs[i * kTL + i];
      const double inv = d != 0.0 ? 1.0 / d : 0.0;
#pragma unroll
      for (int ii = 0; ii < 4; ++ii)
        if (i == bi + ii) {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            x.v[ii][c] *= inv;
            row[bj + c] = x.v[ii][c];
          }
        }
    }
    __syncthreads();
    double rk[4], xr[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      rk[q] = (bi + q < i) ? Rs[(bi + q) * kTL + i] : 0.0;
      xr[q] = row[bj + q];
    }
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int c = 0; c < 4; ++c) x.v[k][c] = fma(-rk[k], xr[c], x.v[k][c]);
  }
  __syncthreads();
}

// X = L^{-1} for unit-lower-triangular L in Ls (forward Gauss-Jordan).
FFB_DEV void inv_unit_lower(const double* Ls, int w, Tile& x, double* buf) {
  const int tid = threadIdx.x, bi = bi_of(tid), bj = bj_of(tid);
  set_identity(x);
  for (int i = 0; i < w; ++i) {
    double* row = buf + (i & 1) * 64;
#pragma unroll
    for (int ii = 0; ii < 4; ++ii)
      if (i == bi + ii) {
#pragma unroll
        for (int c = 0; c < 4; ++c) row[bj + c] = x.v[ii][c];
      }
    __syncthreads();
    double lk[4], xr[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      lk[q] = (bi + q > i && bi + q < w) ? Ls[(bi + q) * kTL + i] : 0.0;
      xr[q] = row[bj + q];
    }
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int c = 0; c < 4; ++c) x.v[k][c] = fma(-lk[k], xr[c], x.v[k][c]);
  }
  __syncthreads();
}

// C = op(A) * op(B) (op = transpose when ta / tb) with A, B in shared memory (kTL).
FFB_DEV void mm(const double* A, const double* B, int w, Tile& c, bool ta = false, bool tb = false) {
  const int tid = threadIdx.x, bi = bi_of(tid), bj = bj_of(tid);
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) c.v[i][j] = 0.0;
  for (int k = 0; k < w; ++k) {
    double a[4], b[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      a[q] = ta ? A[k * kTL + bi + q] : A[(bi + q) * kTL + k];
      b[q] = tb ? B[(bj + q) * kTL + k] : B[k * kTL + bj + q];
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) c.v[i][j] = fma(a[i], b[j], c.v[i][j]);
  }
}

// LU without pivoting of Q_top * D - I with the Householder sign rule (see
// ffb_panel.cu): q tile in, L (unit lower) and U (upper) to Ls/Us, D to Dd.
FFB_DEV void sign_lu(Tile& q, int w, double* Ls, double* Us, double* Dd, double* buf) {
  const int tid = threadIdx.x, bi = bi_of(tid), bj = bj_of(tid);
  for (int t = tid; t < 64 * 64; t += blockDim.x) {
    const int r = t >> 6, c = t & 63;
    Ls[r * kTL + c] = (r == c) ? 1.0 : 0.0;
    Us[r * kTL + c] = 0.0;
  }
  __syncthreads();
  // Steps run four at a time with the in-tile index jj a compile-time constant
  // (c = c4 + jj): the owners of column / row c are the threads with bj == c4 /
  // bi == c4, so publishing a column costs one comparison and four stores
  // instead of a four-way predicated search through the register tile.
  for (int c4 = 0; c4 < w; c4 += 4) {
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      const int c = c4 + jj;
      if (c >= w) break;
      double* col = buf + (jj & 1) * 128;     // column c of the working matrix
      double* rowc = col + 64;                // row c of the working matrix
      if (bj == c4) {
#pragma unroll
        for (int i = 0; i < 4; ++i) col[bi + i] = q.v[i][jj];
      }
      if (bi == c4) {
#pragma unroll
        for (int j = 0; j < 4; ++j) rowc[bj + j] = q.v[jj][j];
      }
      __syncthreads();
      const double z = col[c];
      double d;
      if (fabs(z) == 1.0) d = z > 0.0 ? 1.0 : -1.0;   // identity reflector (tail == 0)
      else d = z > 0.0 ? -1.0 : 1.0;                  // pivot -(1+|z|) = -tau
      const double ucc = d * z - 1.0;
      const double sc = ucc != 0.0 ? d * fast_rcp(ucc) : 0.0;
      if (tid < 64) {
        const int r = tid;
        if (r < c) Us[r * kTL + c] = d * col[r];
        else if (r == c) {
          Us[c * kTL + c] = ucc;
          Dd[c] = d;
        } else if (r < w) {
          Ls[r * kTL + c] = sc * col[r];
        }
      }
      // tiles above or left of block c4 are finished; inside block row / column c4
      // only the rows / columns past c still change
      if (bi >= c4 && bj >= c4) {
        double li[4], rj[4];
#pragma unroll
        for (int q2 = 0; q2 < 4; ++q2) {
          li[q2] = (bi + q2 > c && bi + q2 < w) ? sc * col[bi + q2] : 0.0;
          rj[q2] = (bj + q2 > c && bj + q2 < w) ? rowc[bj + q2] : 0.0;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) q.v[i][j] = fma(-li[i], rj[j], q.v[i][j]);
      }
    }
  }
  __syncthreads();
}


// ---------------------------------------------------------------------------
// Blocked versions (256 threads).  The sequential part of a 64x64 triangular
// inverse is confined to the four 16x16 diagonal blocks, which are inverted
// simultaneously (16 steps, one barrier each: thread t works on block t/64,
// column t%16, rows (t%64)/16 + 4q); the off-diagonal blocks then follow from
// two levels of block products X12 = -X11 A12 X22 (16 -> 32 -> 64).  Entries at
// index >= w are treated as identity.  S: >= 1024 doubles of scratch.

// Off-diagonal blocks of X = U^{-1} from inverted 16x16 diagonal blocks already in
// Xs (strictly lower blocks zero): X12 = -X11 U12 X22, 16 -> 32 -> 64.
FFB_DEV void inv_upper_levels(const double* Us, double* Xs, double* S, int w = 64) {
  const int tid = threadIdx.x;
  // level 1: blocks (0,1) and (2,3): T = U12 X22 (S), X12 = -X11 T; thread -> (k, r, c, c+8)
  // (entries of Us beyond w are zero off the diagonal: callers zero-fill)
  {
    const int k = tid >> 7, e = tid & 127, r = e >> 3, c = e & 7, oo = 32 * k;
    double a0 = 0.0, a1 = 0.0;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const double u = Us[(oo + r) * kTL + oo + 16 + q];
      a0 = fma(u, Xs[(oo + 16 + q) * kTL + oo + 16 + c], a0);
      a1 = fma(u, Xs[(oo + 16 + q) * kTL + oo + 24 + c], a1);
    }
    S[128 + k * 256 + r * 16 + c] = a0;
    S[128 + k * 256 + r * 16 + c + 8] = a1;
    __syncthreads();
    a0 = a1 = 0.0;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const double x = q >= r ? Xs[(oo + r) * kTL + oo + q] : 0.0;
      a0 = fma(x, S[128 + k * 256 + q * 16 + c], a0);
      a1 = fma(x, S[128 + k * 256 + q * 16 + c + 8], a1);
    }
    Xs[(oo + r) * kTL + oo + 16 + c] = -a0;
    Xs[(oo + r) * kTL + oo + 24 + c] = -a1;
    __syncthreads();
  }
  // level 2: T = U12 X22 (32x32, S), X12 = -X11 T; thread -> (r, c + 8 m), m < 4
  // (w <= 32: U12 is identity padding's zero block, so X12 = 0 without the products)
  if (w <= 32) {
    const int r = tid >> 3, c = tid & 7;
#pragma unroll
    for (int m = 0; m < 4; ++m) Xs[r * kTL + 32 + c + 8 * m] = 0.0;
    __syncthreads();
  } else {
    const int r = tid >> 3, c = tid & 7;
    double a[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 8
    for (int q = 0; q < 32; ++q) {
      const double u = Us[r * kTL + 32 + q];
#pragma unroll
      for (int m = 0; m < 4; ++m) a[m] = fma(u, Xs[(32 + q) * kTL + 32 + c + 8 * m], a[m]);
    }
#pragma unroll
    for (int m = 0; m < 4; ++m) S[r * 32 + c + 8 * m] = a[m];
    __syncthreads();
#pragma unroll
    for (int m = 0; m < 4; ++m) a[m] = 0.0;
#pragma unroll 8
    for (int q = 0; q < 32; ++q) {
      const double x = q >= r ? Xs[r * kTL + q] : 0.0;
#pragma unroll
      for (int m = 0; m < 4; ++m) a[m] = fma(x, S[q * 32 + c + 8 * m], a[m]);
    }
#pragma unroll
    for (int m = 0; m < 4; ++m) Xs[r * kTL + 32 + c + 8 * m] = -a[m];
    __syncthreads();
  }
}

// Off-diagonal blocks of X = L^{-1} from inverted 16x16 diagonal blocks already in
// Xs (strictly upper blocks zero): X21 = -X22 L21 X11, 16 -> 32 -> 64.
FFB_DEV void inv_unit_lower_levels(const double* Ls, double* Xs, double* S, int w = 64) {
  const int tid = threadIdx.x;
  // level 1: X21 = -X22 (L21 X11); thread -> (k, r, c, c+8)  (Ls off-diagonal
  // entries beyond w are zero: callers zero-fill)
  {
    const int k = tid >> 7, e = tid & 127, r = e >> 3, c = e & 7, oo = 32 * k;
    double a0 = 0.0, a1 = 0.0;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const double lv = Ls[(oo + 16 + r) * kTL + oo + q];
      a0 = fma(lv, Xs[(oo + q) * kTL + oo + c], a0);
      a1 = fma(lv, Xs[(oo + q) * kTL + oo + c + 8], a1);
    }
    S[128 + k * 256 + r * 16 + c] = a0;
    S[128 + k * 256 + r * 16 + c + 8] = a1;
    __syncthreads();
    a0 = a1 = 0.0;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const double x = q <= r ? Xs[(oo + 16 + r) * kTL + oo + 16 + q] : 0.0;
      a0 = fma(x, S[128 + k * 256 + q * 16 + c], a0);
      a1 = fma(x, S[128 + k * 256 + q * 16 + c + 8], a1);
    }
    Xs[(oo + 16 + r) * kTL + oo + c] = -a0;
    Xs[(oo + 16 + r) * kTL + oo + c + 8] = -a1;
    __syncthreads();
  }
  // level 2: X21 = -X22 (L21 X11) with 32x32 blocks (w <= 32: L21 = 0, X21 = 0)
  if (w <= 32) {
    const int r = tid >> 3, c = tid & 7;
#pragma unroll
    for (int m = 0; m < 4; ++m) Xs[(32 + r) * kTL + c + 8 * m] = 0.0;
    __syncthreads();
  } else {
    const int r = tid >> 3, c = tid & 7;
    double a[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 8
    for (int q = 0; q < 32; ++q) {
      const double lv = Ls[(32 + r) * kTL + q];
#pragma unroll
      for (int m = 0; m < 4; ++m) a[m] = fma(lv, Xs[q * kTL + c + 8 * m], a[m]);
    }
#pragma unroll
    for (int m = 0; m < 4; ++m) S[r * 32 + c + 8 * m] = a[m];
    __syncthreads();
#pragma unroll
    for (int m = 0; m < 4; ++m) a[m] = 0.0;
#pragma unroll 8
    for (int q = 0; q < 32; ++q) {
      const double x = q <= r ? Xs[(32 + r) * kTL + 32 + q] : 0.0;
#pragma unroll
      for (int m = 0; m < 4; ++m) a[m] = fma(x, S[q * 32 + c + 8 * m], a[m]);
    }
#pragma unroll
    for (int m = 0; m < 4; ++m) Xs[(32 + r) * kTL + c + 8 * m] = -a[m];
    __syncthreads();
  }
}

// X = U^{-1} (U upper triangular in Us, kTL), written to Xs (kTL, full 64x64).
// Zero pivots give zero rows (as inv_upper).
FFB_DEV void inv_upper_blk(const double* Us, int w, double* Xs, double* S) {
  const int tid = threadIdx.x, b = tid >> 6, lt = tid & 63, j = lt & 15, i0 = lt >> 4;
  const int o = 16 * b;
  auto uval = [&](int r, int c) -> double {
    if (r >= w || c >= w) return r == c ? 1.0 : 0.0;
    return Us[r * kTL + c];
  };
  double x[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) x[q] = (i0 + 4 * q == j) ? 1.0 : 0.0;
  // zero the strictly lower blocks of X (never written below)
  for (int t = tid; t < 64 * 64; t += blockDim.x) {
    const int r = t >> 6, c = t & 63;
    if ((r >> 4) > (c >> 4)) Xs[r * kTL + c] = 0.0;
  }
  for (int s = 15; s >= 0; --s) {
    double* row = S + (s & 1) * 64;   // [4 blocks][16]
    const double d = uval(o + s, o + s);
    const double inv = d != 0.0 ? 1.0 / d : 0.0;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (i0 + 4 * q == s) {
        x[q] *= inv;
        row[16 * b + j] = x[q];
      }
    __syncthreads();
    const double rs = row[16 * b + j];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = i0 + 4 * q;
      if (i < s) x[q] = fma(-uval(o + i, o + s), rs, x[q]);
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) Xs[(o + i0 + 4 * q) * kTL + o + j] = x[q];
  __syncthreads();
  inv_upper_levels(Us, Xs, S);
}

// X = L^{-1} (L unit lower triangular in Ls, kTL) -> Xs (kTL, full 64x64).
FFB_DEV void inv_unit_lower_blk(const double* Ls, int w, double* Xs, double* S) {
  const int tid = threadIdx.x, b = tid >> 6, lt = tid & 63, j = lt & 15, i0 = lt >> 4;
  const int o = 16 * b;
  auto lval = [&](int r, int c) -> double {
    if (r == c) return 1.0;
    if (r >= w || c >= w) return 0.0;
    return Ls[r * kTL + c];
  };
  double x[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) x[q] = (i0 + 4 * q == j) ? 1.0 : 0.0;
  for (int t = tid; t < 64 * 64; t += blockDim.x) {
    const int r = t >> 6, c = t & 63;
    if ((r >> 4) < (c >> 4)) Xs[r * kTL + c] = 0.0;
  }
  for (int s = 0; s < 16; ++s) {
    double* row = S + (s & 1) * 64;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (i0 + 4 * q == s) row[16 * b + j] = x[q];
    __syncthreads();
    const double rs = row[16 * b + j];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = i0 + 4 * q;
      if (i > s) x[q] = fma(-lval(o + i, o + s), rs, x[q]);
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) Xs[(o + i0 + 4 * q) * kTL + o + j] = x[q];
  __syncthreads();
  inv_unit_lower_levels(Ls, Xs, S);
}

// Upper Cholesky with one barrier per step: the owners of row j of the updated
// Gram publish it (double-buffered), every thread derives the R entries it
// needs itself.  Same contract as chol_upper.
FFB_DEV bool chol_upper1(Tile& g, int w, double* Rs, double* buf) {
  const int tid = threadIdx.x, bi = bi_of(tid), bj = bj_of(tid);
  bool ok = true;
  for (int t = tid; t < 64 * 64; t += blockDim.x) Rs[(t >> 6) * kTL + (t & 63)] = 0.0;
  for (int j = 0; j < w; ++j) {
    double* row = buf + (j & 1) * 64;
#pragma unroll
    for (int ii = 0; ii < 4; ++ii)
      if (j == bi + ii) {
#pragma unroll
        for (int c = 0; c < 4; ++c) row[bj + c] = g.v[ii][c];
      }
    __syncthreads();
    double d = row[j];
    if (!(d > 0.0) || !isfinite(d)) {
      ok = false;
      d = d > 0.0 ? d : 1e-300;
    }
    const double inv = rsqrt(d), rjj = d * inv;
    if (tid < w) Rs[j * kTL + tid] = tid > j ? row[tid] * inv : (tid == j ? rjj : 0.0);
    double rr[4], rc[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      rr[q] = (bi + q > j && bi + q < w) ? row[bi + q] * inv : 0.0;
      rc[q] = (bj + q > j && bj + q < w) ? row[bj + q] * inv : 0.0;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int c = 0; c < 4; ++c) g.v[i][c] = fma(-rr[i], rc[c], g.v[i][c]);
  }
  __syncthreads();
  return ok;
}

// ---------------------------------------------------------------------------
// Blocked right-looking factorizations (256 threads): the sequential chains run
// on 16x16 diagonal blocks inside ONE warp (registers + shuffles, no CTA
// barriers), the off-diagonal block rows and the trailing updates are parallel
// across the CTA.  A 64-wide factorization costs 4 x 3 barriers instead of 64.

// Warp: upper Cholesky of the 16x16 diagonal block at (o, o) of Rs (upper
// triangle holds the updated Gram), in place (strict lower part zeroed), and
// X = R_oo^{-1} into the same block of Xs.  Lane c (< 16) owns column c.
// Columns >= nv are identity padding.  Returns false on a non-positive pivot
// (clamped exactly like chol_upper1).
static __device__ __noinline__ bool warp_chol_inv16(double* Rs, double* Xs, int o, int nv) {
  const int c = threadIdx.x & 31;
  const bool col_ok = c < nv;
  double a[16], dinv[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const double v = Rs[(o + i) * kTL + o + (c & 15)];
    a[i] = col_ok ? (i <= c ? v : 0.0) : (i == c ? 1.0 : 0.0);
  }
  bool ok = true;
  // Right-looking, branch-free: the strict lower part of a[] (rows > c) picks up
  // garbage from the unconditional updates but is never read for the upper
  // factor and is masked on the way out.
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    double d = __shfl_sync(0xffffffffu, a[j], j);
    if (!(d > 0.0) || !isfinite(d)) {
      ok = false;
      d = d > 0.0 ? d : 1e-300;
    }
    const double inv = rsqrt(d);
    dinv[j] = inv;
    a[j] = (c == j) ? d * inv : a[j] * inv;
#pragma unroll
    for (int i = j + 1; i < 16; ++i) a[i] = fma(-__shfl_sync(0xffffffffu, a[j], i), a[j], a[i]);
  }
  // X = R^{-1}, column c: x_s = (delta_sc - sum_{k>s} R_sk x_k) / R_ss, 1/R_ss = dinv[s]
  // (x_k = 0 for k > c, so lower garbage in other lanes' a[] never contributes)
  double x[16];
#pragma unroll
  for (int s = 15; s >= 0; --s) {
    double acc0 = (c == s) ? 1.0 : 0.0, acc1 = 0.0;
#pragma unroll
    for (int k = s + 1; k < 16; ++k) {
      const double rsk = __shfl_sync(0xffffffffu, a[s], k);
      if ((k - s) & 1) acc0 = fma(-rsk, x[k], acc0);
      else acc1 = fma(-rsk, x[k], acc1);
    }
    x[s] = (acc0 + acc1) * dinv[s];
  }
  if (c < 16) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      Rs[(o + i) * kTL + o + c] = i <= c ? a[i] : 0.0;
      Xs[(o + i) * kTL + o + c] = x[i];
    }
  }
  return ok;
}

// Upper Cholesky R^T R = G (tile in, upper triangle used) and X = R^{-1}:
// R -> Rs (full 64x64, zeros outside the w x w upper triangle), X -> Xs (full
// 64x64, identity beyond w, zero pivots give zero rows).  Same contract as
// chol_upper1 followed by inv_upper_blk.  S: >= 1024 doubles of scratch.
FFB_DEV bool chol_inv_blk(Tile& g, int w, double* Rs, double* Xs, double* S) {
  __shared__ int s_ok;
  const int tid = threadIdx.x, bi = bi_of(tid), bj = bj_of(tid), warp = tid >> 5;
  const int nbk = (w + 15) >> 4;
  for (int t = tid; t < 64 * 64; t += blockDim.x) {
    const int r = t >> 6, c = t & 63;
    Rs[r * kTL + c] = 0.0;
    Xs[r * kTL + c] = (r == c && (r >> 4) >= nbk) ? 1.0 : 0.0;
  }
  if (tid == 0) s_ok = 1;
  __syncthreads();
  for (int K = 0; K < nbk; ++K) {
    const int o = 16 * K, e = o + 16, ncol = w - e;
    // publish block row K of the updated Gram (upper part)
    if ((bi >> 4) == K && bj + 3 >= o) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (bj + j >= bi + i && bj + j < w) Rs[(bi + i) * kTL + bj + j] = g.v[i][j];
    }
    __syncthreads();
    if (warp == 0) {
      const bool ok = warp_chol_inv16(Rs, Xs, o, w - o < 16 ? w - o : 16);
      if (!ok && (tid & 31) == 0) s_ok = 0;
    }
    __syncthreads();
    if (ncol <= 0) break;
    // R_KJ = R_KK^{-T} G_KJ = X_KK^T G_KJ  -> S (16 x 64)
    for (int t = tid; t < 16 * ncol; t += blockDim.x) {
      const int i = t & 15, cc = e + (t >> 4);
      double a0 = 0.0, a1 = 0.0;
#pragma unroll
      for (int k = 0; k < 16; k += 2) {
        if (k <= i) a0 = fma(Xs[(o + k) * kTL + o + i], Rs[(o + k) * kTL + cc], a0);
        if (k + 1 <= i) a1 = fma(Xs[(o + k + 1) * kTL + o + i], Rs[(o + k + 1) * kTL + cc], a1);
      }
      S[i * 64 + cc] = a0 + a1;
    }
    __syncthreads();
    for (int t = tid; t < 16 * ncol; t += blockDim.x) {
      const int i = t & 15, cc = e + (t >> 4);
      Rs[(o + i) * kTL + cc] = S[i * 64 + cc];
    }
    // trailing update of the upper Gram: G_ab -= sum_k R_ka R_kb (a, b >= e)
    if (bi >= e && bj + 3 >= bi && bi < w && bj < w) {
#pragma unroll 4
      for (int k = 0; k < 16; ++k) {
        double ra[4], rb[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          ra[q] = bi + q < w ? S[k * 64 + bi + q] : 0.0;
          rb[q] = bj + q < w ? S[k * 64 + bj + q] : 0.0;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) g.v[i][j] = fma(-ra[i], rb[j], g.v[i][j]);
      }
    }
    __syncthreads();
  }
  // R beyond w: padding columns of the last block hold identity -> zero
  for (int t = tid; t < 64; t += blockDim.x)
    if (t >= w) Rs[t * kTL + t] = 0.0;
  const bool ok = s_ok != 0;
  __syncthreads();
  inv_upper_levels(Rs, Xs, S, w);
  return ok;
}

// LU without pivoting of Q_top * D - I with the Householder sign rule (same
// arithmetic contract as sign_lu), blocked: L (unit lower) -> Ls, U (upper,
// column-scaled by D) -> Us, D -> Dd, and the inverses U^{-1} -> Ui, L^{-1} -> Li
// (same contract as inv_upper_blk / inv_unit_lower_blk).  S: >= 1024 doubles.
// U^{-1} (Us upper, zero pivots -> zero rows) into Ui and L^{-1} (Ls unit lower)
// into Li together: the eight 16x16 diagonal-block inverses run one per warp
// from shared memory (no CTA barriers), then the block-product levels.  Same
// contract as inv_upper_blk + inv_unit_lower_blk.  S: >= 1024 doubles.
FFB_DEV void inv_upper_lower_blk(const double* Us, const double* Ls, int w, double* Ui, double* Li,
                                 double* S) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int t = tid; t < 64 * 64; t += blockDim.x) {
    const int r = t >> 6, c = t & 63;
    if ((r >> 4) > (c >> 4)) Ui[r * kTL + c] = 0.0;
    if ((r >> 4) < (c >> 4)) Li[r * kTL + c] = 0.0;
  }
  {
    const int o = 16 * (warp & 3), c = lane & 15;
    double x[16];
    if (warp < 4) {
      auto uval = [&](int r, int k) -> double {
        if (o + r >= w || o + k >= w) return r == k ? 1.0 : 0.0;
        return Us[(o + r) * kTL + o + k];
      };
#pragma unroll
      for (int s = 15; s >= 0; --s) {
        double acc0 = (c == s) ? 1.0 : 0.0, acc1 = 0.0;
#pragma unroll
        for (int k = s + 1; k < 16; ++k) {
          if ((k - s) & 1) acc0 = fma(-uval(s, k), x[k], acc0);
          else acc1 = fma(-uval(s, k), x[k], acc1);
        }
        const double d = uval(s, s);
        x[s] = (acc0 + acc1) * (d != 0.0 ? 1.0 / d : 0.0);
      }
      if (lane < 16)
#pragma unroll
        for (int i = 0; i < 16; ++i) Ui[(o + i) * kTL + o + c] = x[i];
    } else {
      auto lval = [&](int r, int k) -> double {
        if (r == k) return 1.0;
        if (o + r >= w || o + k >= w) return 0.0;
        return Ls[(o + r) * kTL + o + k];
      };
#pragma unroll
      for (int s = 0; s < 16; ++s) {
        double acc0 = (c == s) ? 1.0 : 0.0, acc1 = 0.0;
#pragma unroll
        for (int k = 0; k < s; ++k) {
          if ((s - k) & 1) acc0 = fma(-lval(s, k), x[k], acc0);
          else acc1 = fma(-lval(s, k), x[k], acc1);
        }
        x[s] = acc0 + acc1;
      }
      if (lane < 16)
#pragma unroll
        for (int i = 0; i < 16; ++i) Li[(o + i) * kTL + o + c] = x[i];
    }
  }
  __syncthreads();
  inv_upper_levels(Us, Ui, S, w);
  inv_unit_lower_levels(Ls, Li, S, w);
}

}  // namespace tile64
}  // namespace ffb
