// FP64 tensor-core GEMM engine: C = alpha * op(A) op(B) + beta * C on sm_100a DMMA
// (mma.sync.m8n8k4.f64 -> DMMA.8x8x4; tcgen05 has no f64 kind).
//
// Operand addressing (column-major storage everywhere):
//   A(i,k) = A_KC ? A[k + i*lda] : A[i + k*lda]      (i < M, k < K)
//   B(k,j) = B_KC ? B[k + j*ldb] : B[j + k*ldb]      (k < K, j < N)
//   C(i,j) = C[i + j*ldc]
// Tiles are staged global->shared with a multi-stage cp.async pipeline, each
// operand kept in shared memory along its contiguous global dimension and
// padded so that DMMA fragment loads are bank-conflict free.  Split-K writes
// fp64 partial tiles that a second kernel reduces in fixed order, so results
// are bitwise deterministic run to run.
#pragma once
#include "ffb_common.cuh"

namespace ffb {

struct GemmArgs {
  int64_t M, N, K;
  double alpha, beta;
  const double* A;
  int64_t lda;
  const double* B;
  int64_t ldb;
  double* C;
  int64_t ldc;
  double* partial;   // split-K scratch: splits * M * N doubles (ld = M)
  int splits;
  int force_partial; // write partial tiles even when splits == 1
  int64_t k_per;     // K range per split (multiple of BK)
};

template <int BM, int BK>
struct APad {
  static constexpr int kc = BK + ((4 - BK % 16) + 16) % 16;        // (BK+pad) % 16 == 4
  static constexpr int mc = BM + ((8 - BM % 16) + 16) % 16;        // (BM+pad) % 16 == 8
};

template <int BM, int BN, int BK, int WM, int WN, bool A_KC, bool B_KC, int STAGES>
struct GemmCfg {
  static constexpr int kWarpsM = BM / WM, kWarpsN = BN / WN;
  static constexpr int kThreads = 32 * kWarpsM * kWarpsN;
  static constexpr int kTM = WM / 8, kTN = WN / 8;
  static constexpr int kAStage = A_KC ? BM * APad<BM, BK>::kc : BK * APad<BM, BK>::mc;
  static constexpr int kBStage = B_KC ? BN * APad<BN, BK>::kc : BK * APad<BN, BK>::mc;
  static constexpr size_t kSmem = sizeof(double) * (size_t)STAGES * (kAStage + kBStage);
};

// Operand tile loader: each thread owns a fixed set of (row, k) slots of the
// tile; global pointers and shared offsets are computed once and advanced by a
// constant per k-tile.  VEC2: 16-byte cp.async pairs along the contiguous
// dimension (requires 16-byte aligned base and even leading dimension).
template <int R, int BK, bool KC, bool VEC2, int NT>
struct TileLoader {
  // elements (or pairs) per thread
  static constexpr int kUnits = (R * BK) / (VEC2 ? 2 : 1);
  static constexpr int kPer = (kUnits + NT - 1) / NT;
  static constexpr int LD = KC ? APad<R, BK>::kc : APad<R, BK>::mc;
  const double* g[kPer];
  uint32_t soff[kPer];
  int kk[kPer];      // k index inside the tile of the unit's first element
  int rr[kPer];      // row (M or N) index of the unit (first element)
  bool live[kPer];

  FFB_DEV void init(const double* base, int64_t ld, int64_t r0, int64_t rows, int64_t k0, int tid) {
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int idx = tid + u * NT;
      live[u] = idx < kUnits;
      int r, k;
      if (KC) {   // k contiguous: units run along k
        constexpr int kpr = VEC2 ? BK / 2 : BK;
        r = idx / kpr;
        k = (idx % kpr) * (VEC2 ? 2 : 1);
      } else {    // row contiguous: units run along rows
        constexpr int rpk = VEC2 ? R / 2 : R;
        k = idx / rpk;
        r = (idx % rpk) * (VEC2 ? 2 : 1);
      }
      rr[u] = r;
      kk[u] = k;
      const int64_t gr = r0 + r;
      live[u] = live[u] && gr < rows;
      g[u] = base + (live[u] ? (KC ? (k0 + k) + gr * ld : gr + (k0 + k) * ld) : 0);
      soff[u] = KC ? (uint32_t)(r * LD + k) : (uint32_t)(k * LD + r);
    }
  }
  // kvalid: number of valid k in this tile (BK except the K tail); rows: bound
  FFB_DEV void load(double* smem, int kvalid, int64_t r0, int64_t rows, int64_t ld) {
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      if (u * NT + (int)threadIdx.x >= kUnits) continue;
      double* dst = smem + soff[u];
      if (VEC2) {
        int bytes = 0;
        if (live[u]) {
          if (KC) {
            bytes = kk[u] + 1 < kvalid ? 16 : (kk[u] < kvalid ? 8 : 0);
          } else {
            bytes = kk[u] < kvalid ? (r0 + rr[u] + 1 < rows ? 16 : 8) : 0;
          }
        }
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)),
                     "l"(bytes ? g[u] : g[0]), "r"(bytes));
      } else {
        const bool ok = live[u] && kk[u] < kvalid;
        cp_async8(dst, ok ? g[u] : g[0], ok);
      }
    }
    (void)ld;
  }
  FFB_DEV void advance(int64_t ld) {
#pragma unroll
    for (int u = 0; u < kPer; ++u) g[u] += KC ? BK : (int64_t)BK * ld;
  }
};

template <int BM, int BN, int BK, int WM, int WN, bool A_KC, bool B_KC, int STAGES, bool VEC2>
__global__ void __launch_bounds__(GemmCfg<BM, BN, BK, WM, WN, A_KC, B_KC, STAGES>::kThreads)
    gemm_f64_kernel(GemmArgs g) {
  using Cfg = GemmCfg<BM, BN, BK, WM, WN, A_KC, B_KC, STAGES>;
  constexpr int NT = Cfg::kThreads;
  constexpr int ALD = A_KC ? APad<BM, BK>::kc : APad<BM, BK>::mc;
  constexpr int BLD = B_KC ? APad<BN, BK>::kc : APad<BN, BK>::mc;
  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + STAGES * Cfg::kAStage;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm0 = (warp / Cfg::kWarpsN) * WM, wn0 = (warp % Cfg::kWarpsN) * WN;
  const int64_t i0 = (int64_t)blockIdx.y * BM, j0 = (int64_t)blockIdx.x * BN;
  const int split = blockIdx.z;
  const int64_t kbeg = (int64_t)split * g.k_per;
  const int64_t kend = min(g.K, kbeg + g.k_per);
  const int nk = kbeg < kend ? (int)((kend - kbeg + BK - 1) / BK) : 0;

  TileLoader<BM, BK, A_KC, VEC2, NT> la;
  TileLoader<BN, BK, B_KC, VEC2, NT> lb;
  la.init(g.A, g.lda, i0, g.M, kbeg, tid);
  lb.init(g.B, g.ldb, j0, g.N, kbeg, tid);

  double acc[Cfg::kTM][Cfg::kTN][2];
#pragma unroll
  for (int a = 0; a < Cfg::kTM; ++a)
#pragma unroll
    for (int b = 0; b < Cfg::kTN; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  int fetched = 0;
  auto fetch = [&](int stage) {
    const int64_t k0 = kbeg + (int64_t)fetched * BK;
    const int64_t krem = kend - k0;
    const int kvalid = krem < BK ? (int)krem : BK;
    la.load(As + stage * Cfg::kAStage, kvalid, i0, g.M, g.lda);
    lb.load(Bs + stage * Cfg::kBStage, kvalid, j0, g.N, g.ldb);
    la.advance(g.lda);
    lb.advance(g.ldb);
    ++fetched;
  };

#pragma unroll
  for (int st = 0; st < STAGES - 1; ++st) {
    if (st < nk) fetch(st);
    cp_async_commit();
  }

  const int fr = lane >> 2, fk = lane & 3;
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int pf = kt + STAGES - 1;
      if (pf < nk) fetch(pf % STAGES);
      cp_async_commit();
    }
    const double* as = As + (kt % STAGES) * Cfg::kAStage;
    const double* bs = Bs + (kt % STAGES) * Cfg::kBStage;
#pragma unroll
    for (int k4 = 0; k4 < BK; k4 += 4) {
      double af[Cfg::kTM], bf[Cfg::kTN];
#pragma unroll
      for (int a = 0; a < Cfg::kTM; ++a) {
        const int r = wm0 + a * 8 + fr, kk = k4 + fk;
        af[a] = A_KC ? as[r * ALD + kk] : as[kk * ALD + r];
      }
#pragma unroll
      for (int b = 0; b < Cfg::kTN; ++b) {
        const int c = wn0 + b * 8 + fr, kk = k4 + fk;
        bf[b] = B_KC ? bs[c * BLD + kk] : bs[kk * BLD + c];
      }
#pragma unroll
      for (int a = 0; a < Cfg::kTM; ++a)
#pragma unroll
        for (int b = 0; b < Cfg::kTN; ++b) dmma_884(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
    }
  }
  cp_async_wait<0>();

  // Epilogue.
#pragma unroll
  for (int a = 0; a < Cfg::kTM; ++a) {
    const int64_t gi = i0 + wm0 + a * 8 + fr;
    if (gi >= g.M) continue;
#pragma unroll
    for (int b = 0; b < Cfg::kTN; ++b) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t gj = j0 + wn0 + b * 8 + 2 * fk + h;
        if (gj >= g.N) continue;
        if (g.splits == 1 && !g.force_partial) {
          double* cp = g.C + gi + gj * g.ldc;
          const double v = g.alpha * acc[a][b][h];
          *cp = g.beta == 0.0 ? v : v + g.beta * (*cp);
        } else {
          g.partial[(size_t)split * g.M * g.N + gi + gj * g.M] = acc[a][b][h];
        }
      }
    }
  }
}

// Fixed-order reduction of split-K partials into C.
__global__ void gemm_splitk_reduce(const double* __restrict__ part, int splits, int64_t M, int64_t N,
                                   double alpha, double beta, double* C, int64_t ldc) {
  const int64_t total = M * N;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < splits; ++q) s += part[(size_t)q * total + t];
    const int64_t i = t % M, j = t / M;
    double* cp = C + i + j * ldc;
    const double v = alpha * s;
    *cp = beta == 0.0 ? v : v + beta * (*cp);
  }
}

}  // namespace ffb
