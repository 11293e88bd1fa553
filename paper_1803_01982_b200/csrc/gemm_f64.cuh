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

template <int BM, int BN, int BK, int WM, int WN, bool A_KC, bool B_KC, int STAGES>
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

  auto load_tile = [&](int stage, int64_t k0) {
    double* as = As + stage * Cfg::kAStage;
    double* bs = Bs + stage * Cfg::kBStage;
#pragma unroll 4
    for (int idx = tid; idx < BM * BK; idx += NT) {
      int i, kk;
      if (A_KC) { kk = idx % BK; i = idx / BK; } else { i = idx % BM; kk = idx / BM; }
      const int64_t gi = i0 + i, gk = k0 + kk;
      const bool ok = gi < g.M && gk < kend;
      const double* src = g.A + (ok ? (A_KC ? gk + gi * g.lda : gi + gk * g.lda) : 0);
      cp_async8(as + (A_KC ? i * ALD + kk : kk * ALD + i), src, ok);
    }
#pragma unroll 4
    for (int idx = tid; idx < BN * BK; idx += NT) {
      int j, kk;
      if (B_KC) { kk = idx % BK; j = idx / BK; } else { j = idx % BN; kk = idx / BN; }
      const int64_t gj = j0 + j, gk = k0 + kk;
      const bool ok = gj < g.N && gk < kend;
      const double* src = g.B + (ok ? (B_KC ? gk + gj * g.ldb : gj + gk * g.ldb) : 0);
      cp_async8(bs + (B_KC ? j * BLD + kk : kk * BLD + j), src, ok);
    }
  };

  double acc[Cfg::kTM][Cfg::kTN][2];
#pragma unroll
  for (int a = 0; a < Cfg::kTM; ++a)
#pragma unroll
    for (int b = 0; b < Cfg::kTN; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) load_tile(s, kbeg + (int64_t)s * BK);
    cp_async_commit();
  }

  const int fr = lane >> 2, fk = lane & 3;
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int pf = kt + STAGES - 1;
      if (pf < nk) load_tile(pf % STAGES, kbeg + (int64_t)pf * BK);
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
