// Host dispatcher for the FP64 DMMA GEMM engine (tile configs x operand layouts).
#include <algorithm>
#include <cstdlib>
#include <cstdio>

#include <cudaTypedefs.h>

#include <mutex>

#include "ffb_gemm.h"
#include "gemm_f64.cuh"

namespace ffb {

namespace {

template <int BM, int BN, int BK, int WM, int WN, bool AK, bool BKC, int ST, bool V2, bool SK,
          bool TMA = false>
cudaError_t launch_cfg2(cudaStream_t st, const GemmArgs& g, dim3 grid) {
  using Cfg = GemmCfg<BM, BN, BK, WM, WN, AK, BKC, ST, TMA>;
  auto kern = gemm_f64_kernel<BM, BN, BK, WM, WN, AK, BKC, ST, V2, SK, TMA>;
  static std::atomic<unsigned long long> attr{0};
  ensure_smem_optin((const void*)kern, (int)Cfg::kSmem, attr);
  kern<<<grid, Cfg::kThreads, Cfg::kSmem, st>>>(g);
  return cudaGetLastError();
}

template <int BM, int BN, int BK, int WM, int WN, bool AK, bool BKC, int ST, bool V2>
cudaError_t launch_cfg1(cudaStream_t st, const GemmArgs& g, dim3 grid) {
  if (g.sk_per > 0) return launch_cfg2<BM, BN, BK, WM, WN, AK, BKC, ST, V2, true>(st, g, grid);
  return launch_cfg2<BM, BN, BK, WM, WN, AK, BKC, ST, V2, false>(st, g, grid);
}

// resident CTAs per SM of a tile config (cached)
template <int BM, int BN, int BK, int WM, int WN, int ST>
int occupancy() {
  static int occ = 0;
  if (!occ) {
    using Cfg = GemmCfg<BM, BN, BK, WM, WN, true, true, ST>;
    auto kern = gemm_f64_kernel<BM, BN, BK, WM, WN, true, true, ST, true, true>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::kSmem);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, Cfg::kThreads, Cfg::kSmem) != cudaSuccess || occ < 1)
      occ = 1;
  }
  return occ;
}

int occupancy_of(int cfg) {
  switch (cfg) {
    case 0: return occupancy<48, 64, 16, 24, 32, 4>();
    case 1: return occupancy<64, 64, 16, 32, 32, 4>();
    case 2: return occupancy<96, 64, 16, 48, 32, 4>();
    case 3: return occupancy<128, 64, 16, 32, 32, 3>();
    case 4: return occupancy<128, 96, 16, 32, 48, 3>();
    case 5: return occupancy<16, 64, 16, 16, 16, 4>();
    case 6: return occupancy<32, 64, 16, 16, 32, 4>();
    case 7: return occupancy<32, 32, 16, 16, 16, 4>();
    case 8: return occupancy<64, 288, 16, 32, 72, 3>();
    case 9: return occupancy<64, 144, 16, 32, 72, 3>();
    case 11: return occupancy<80, 64, 16, 40, 32, 4>();
    default: return occupancy<64, 216, 16, 32, 72, 3>();
  }
}

// 16-byte pair loads need 16-byte aligned bases and even leading dimensions
inline bool vec2_ok(const GemmArgs& g) {
  auto al = [](const void* p) { return ((uintptr_t)p & 15u) == 0; };
  return al(g.A) && al(g.B) && (g.lda % 2 == 0) && (g.ldb % 2 == 0) && (g.k_per % 2 == 0);
}

template <int BM, int BN, int BK, int WM, int WN, bool AK, bool BKC, int ST>
cudaError_t launch_cfg(cudaStream_t st, const GemmArgs& g, dim3 grid) {
  if (vec2_ok(g)) return launch_cfg1<BM, BN, BK, WM, WN, AK, BKC, ST, true>(st, g, grid);
  return launch_cfg1<BM, BN, BK, WM, WN, AK, BKC, ST, false>(st, g, grid);
}

template <int BM, int BN, int WM, int WN, int ST>
cudaError_t launch_tma_cfg(cudaStream_t st, const GemmArgs& g, dim3 grid) {
  if (g.sk_per > 0) return launch_cfg2<BM, BN, 16, WM, WN, true, true, ST, true, true, true>(st, g, grid);
  return launch_cfg2<BM, BN, 16, WM, WN, true, true, ST, true, false, true>(st, g, grid);
}

// TMA-staged tiles for the k-contiguous x k-contiguous products (the sketch
// Omega A, the WT rows Y^T A): configs with a TMA instance
bool tma_cfg(int cfg) { return cfg == 0 || cfg == 1 || cfg == 2 || cfg == 5 || cfg == 6 || cfg == 11; }

cudaError_t launch_tma(int cfg, cudaStream_t st, const GemmArgs& g, dim3 grid) {
  switch (cfg) {
    case 0: return launch_tma_cfg<48, 64, 24, 32, 4>(st, g, grid);
    case 1: return launch_tma_cfg<64, 64, 32, 32, 4>(st, g, grid);
    case 2: return launch_tma_cfg<96, 64, 48, 32, 4>(st, g, grid);
    case 5: return launch_tma_cfg<16, 64, 16, 16, 4>(st, g, grid);
    case 6: return launch_tma_cfg<32, 64, 16, 32, 4>(st, g, grid);
    default: return launch_tma_cfg<80, 64, 40, 32, 4>(st, g, grid);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 tma_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// (K inner, rows) k-contiguous operand with leading dimension ld, box (16, box_rows)
bool encode_kc(CUtensorMap* map, const double* base, int64_t K, int64_t rows, int64_t ld, int box_rows) {
  auto enc = tma_encoder();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(double)};
  cuuint32_t box[2] = {16u, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1u, 1u};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

struct Shape {
  int bm, bn, bk;
};

// Tile selection by M (the output rows): sketch / WT rows have M = s or b <= 96,
// the tall products (A*Yhat, panel updates) have M = m.
int pick_cfg(int64_t M, int64_t N, int64_t K) {
  static int forced = -2;
  if (forced == -2) {
    const char* e = getenv("FFB_GEMM_CFG");
    forced = e ? atoi(e) : -1;
  }
  if (forced >= 0) return forced > 11 ? 11 : forced;
  if (M <= 16) return 5;
  // small outputs with short K (no split-K to fill the GPU): 32 x 32 tiles so the
  // work spreads over many SMs instead of a few large tiles
  const int64_t tiles64 = ((M + 63) / 64) * ((N + 63) / 64);
  static int smallk = -2;  // FFB_GEMM_SMALL: tile config of small short-K products (tuning)
  if (smallk == -2) {
    const char* e = getenv("FFB_GEMM_SMALL");
    smallk = e ? atoi(e) : 7;
  }
  if (tiles64 < 148 && K < 1024) return smallk;
  if (M <= 32) return 6;
  if (M <= 48) return 0;
  if (M <= 64) return 1;
  static int m80 = -2;   // FFB_GEMM_M80: tile config of 64 < M <= 80 (the sketch, s = 80)
  if (m80 == -2) {
    const char* e = getenv("FFB_GEMM_M80");
    m80 = e ? atoi(e) : 11;
  }
  if (M <= 80) return m80;
  if (M <= 96) return 2;
  static int tallk = -2;   // FFB_GEMM_TALLK: tile config of tall short-K products (tuning)
  if (tallk == -2) {
    const char* e = getenv("FFB_GEMM_TALLK");
    tallk = e ? atoi(e) : 0;
  }
  if (M >= 1024 && K < 512) return tallk;   // tall, short K: many small tiles fill the SMs
  // (configs 8 and 10 -- one wide N tile per row block, the big operand read from
  // HBM once -- and 128 x 144 / 64 x 128 tiles measured slower than 64 x 144)
  if (M >= 1024 && N > 192) return 9;   // tall, wide N (A*Yhat at l = 272 / 420): 64 x 144
                                       // tiles + stream-K: 28.4 / 30.1 TF vs 25.5 / 23.7 (128 x 96)
  // N just under one 144-column tile (cfg5's A*Yhat, l = 144): 64 x 144 tiles with
  // no padding columns, 20.8 TF against 16.7 on 128 x 64 (a quarter of the third
  // N tile empty)
  if (M >= 1024 && N > 128 && N <= 144 && K >= 1024) return 9;
  if (M >= 1024) {
    // tall products (N = l): pick the N tile with less padding waste
    const int64_t w64 = (N + 63) / 64 * 64 - N, w96 = (N + 95) / 96 * 96 - N;
    return (N > 64 && w96 < w64) ? 4 : 3;
  }
  return 1;
}

const Shape kShapes[12] = {{48, 64, 16},  {64, 64, 16}, {96, 64, 16},  {128, 64, 16},
                           {128, 96, 16}, {16, 64, 16}, {32, 64, 16},  {32, 32, 16},
                           {64, 288, 16}, {64, 144, 16}, {64, 216, 16}, {80, 64, 16}};

template <bool AK, bool BKC>
cudaError_t launch_layout(int cfg, cudaStream_t st, const GemmArgs& g, dim3 grid) {
  switch (cfg) {
    case 0: return launch_cfg<48, 64, 16, 24, 32, AK, BKC, 4>(st, g, grid);
    case 1: return launch_cfg<64, 64, 16, 32, 32, AK, BKC, 4>(st, g, grid);
    case 2: return launch_cfg<96, 64, 16, 48, 32, AK, BKC, 4>(st, g, grid);
    case 3: return launch_cfg<128, 64, 16, 32, 32, AK, BKC, 3>(st, g, grid);
    case 4: return launch_cfg<128, 96, 16, 32, 48, AK, BKC, 3>(st, g, grid);
    case 5: return launch_cfg<16, 64, 16, 16, 16, AK, BKC, 4>(st, g, grid);
    case 6: return launch_cfg<32, 64, 16, 16, 32, AK, BKC, 4>(st, g, grid);
    case 7: return launch_cfg<32, 32, 16, 16, 16, AK, BKC, 4>(st, g, grid);
    case 8: return launch_cfg<64, 288, 16, 32, 72, AK, BKC, 3>(st, g, grid);
    case 9: return launch_cfg<64, 144, 16, 32, 72, AK, BKC, 3>(st, g, grid);
    case 11: return launch_cfg<80, 64, 16, 40, 32, AK, BKC, 4>(st, g, grid);
    default: return launch_cfg<64, 216, 16, 32, 72, AK, BKC, 3>(st, g, grid);
  }
}

}  // namespace

cudaError_t gemm_f64(GemmCtx& c, cudaStream_t st, int64_t M, int64_t N, int64_t K, double alpha,
                     const double* A, int64_t lda, bool akc, const double* B, int64_t ldb, bool bkc,
                     double beta, double* C, int64_t ldc, GemmPartialOut* pout) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  const int cfg = pick_cfg(M, N, K);
  static int glog = -1;
  if (glog < 0) glog = getenv("FFB_GEMM_LOG") ? 1 : 0;
  if (glog) fprintf(stderr, "[gemm] M=%lld N=%lld K=%lld akc=%d bkc=%d cfg=%d\n", (long long)M, (long long)N,
                    (long long)K, (int)akc, (int)bkc, cfg);
  const Shape sh = kShapes[cfg];
  int64_t gx = (N + sh.bn - 1) / sh.bn, gy = (M + sh.bm - 1) / sh.bm;
  const int64_t tiles = gx * gy;
  const int64_t target = 2LL * c.sms;
  int64_t splits = 1;
  if (K <= 0) {
    splits = 1;
  } else if (pout) {
    splits = std::max<int64_t>(1, std::min<int64_t>(pout->max_splits, K / 256));
    while (splits > 1 && (size_t)splits * M * N > c.partial_cap) --splits;
  } else if (tiles < target) {
    splits = (target + tiles - 1) / tiles;
    splits = std::min<int64_t>(splits, std::max<int64_t>(1, K / (sh.bk * 8)));
    splits = std::min<int64_t>(splits, 64);
    while (splits > 1 && (size_t)splits * M * N > c.partial_cap) --splits;
  }
  GemmArgs g;
  g.M = M;
  g.N = N;
  g.K = K;
  g.alpha = alpha;
  g.beta = beta;
  g.A = A;
  g.lda = lda;
  g.B = B;
  g.ldb = ldb;
  g.C = C;
  g.ldc = ldc;
  g.partial = c.partial;
  g.splits = (int)splits;
  g.force_partial = pout ? 1 : 0;
  g.sk_per = 0;
  g.sk_maxseg = 0;
  g.sk_tiles_n = (int)gx;
  g.sk_lock = 0;
  g.sk_kiters = (K + sh.bk - 1) / sh.bk;
  g.sk_cnt = nullptr;
  int64_t kper = (K + splits - 1) / splits;
  kper = ((kper + sh.bk - 1) / sh.bk) * sh.bk;
  g.k_per = std::max<int64_t>(kper, sh.bk);
  if (K > 0) {
    // recompute the effective split count after rounding k_per up
    splits = (K + g.k_per - 1) / g.k_per;
    g.splits = (int)splits;
  }
  if (pout) {
    pout->part = c.partial;
    pout->splits = (int)splits;
  }
  if (K <= 0) {
    // C = beta * C (alpha * 0): handled by a tile pass with empty K.
    g.splits = 1;
    g.force_partial = pout ? 1 : 0;
  }
  // Stream-K (persistent, equal iteration ranges, deterministic fixup) whenever the
  // classic grid would leave SMs idle: removes split-K wave quantisation.
  bool use_sk = false;
  static int sk_mode = -2;   // FFB_GEMM_SK: 0 = never, 1 = auto (default)
  if (sk_mode == -2) {
    const char* e = getenv("FFB_GEMM_SK");
    sk_mode = e ? atoi(e) : 1;
  }
  if (!pout && K > 0 && sk_mode != 0) {
    const int64_t slots = (int64_t)c.sms * occupancy_of(cfg);
    const int64_t kit = g.sk_kiters;
    const int64_t waves = (tiles + slots - 1) / slots;
    const double eff = (double)tiles / (double)(waves * slots);
    // short K: the fixup would cost more than the tail it removes
    if (eff < 0.9 && kit >= 32 && tiles >= 32) {
      // Lockstep over N: a row operand larger than L2 with 2-4 N tiles (A*Yhat at
      // l = 272 / 420) was streamed from HBM once per N tile, because the CTAs on
      // the N tiles of one row block worked at different k offsets; here the tn
      // CTAs of a range owner walk the same (row block, k) range together
      // (FFB_GEMM_LOCK=0 disables)
      const char* lock_env = getenv("FFB_GEMM_LOCK");   // read per call (tests toggle it)
      const bool lock = !(lock_env && atoi(lock_env) == 0) && gx >= 2 && gx <= 4 && (double)M * (double)K * 8.0 > 96e6;
      const int64_t tn = lock ? gx : 1;
      const int64_t rtiles = tiles / tn;          // tiles of the range space
      const int64_t total = rtiles * kit;
      // <= 8 CTAs cover any tile (bounded fixup work), >= 4 k-tiles per CTA
      int64_t G = std::min<int64_t>(std::min<int64_t>(slots / tn, rtiles * 8), std::max<int64_t>(1, total / 4));
      G = std::max<int64_t>(G, 1);
      int64_t per = (total + G - 1) / G;
      G = (total + per - 1) / per;
      const int64_t maxseg = (per + kit - 1) / kit + 1;
      if ((size_t)(G * tn) * maxseg * sh.bm * sh.bn <= c.partial_cap && c.counters &&
          tiles <= (int64_t)c.counter_cap && kit / per + 2 <= 16) {
        use_sk = true;
        g.sk_per = per;
        g.sk_cnt = c.counters;
        g.sk_maxseg = (int)maxseg;
        g.sk_lock = lock ? 1 : 0;
        g.splits = 1;
        gx = G * tn;
        gy = 1;
      }
    }
  }
  // TMA staging for k-contiguous x k-contiguous products (FFB_GEMM_TMA=0 disables)
  static int tma_mode = -2;
  if (tma_mode == -2) {
    const char* e = getenv("FFB_GEMM_TMA");
    tma_mode = e ? atoi(e) : 1;
  }
  auto al16 = [](const void* p) { return ((uintptr_t)p & 15u) == 0; };
  // measured (tools/gemm_bench.py): TMA wins on the wide products (>= ~100 output
  // tiles: cfg2 sketch 29.7 -> 31.1 TF, WT 25.8 -> 27.8 TF) and loses on the
  // few-tile stream-K ones (cfg3 / cfg5 WT), which keep cp.async
  const bool use_tma = tma_mode != 0 && akc && bkc && tma_cfg(cfg) && K >= 256 &&
                       (tma_mode == 2 || tiles >= 96) && al16(A) && al16(B) &&
                       lda % 2 == 0 && ldb % 2 == 0 && M < (1LL << 31) && N < (1LL << 31) &&
                       K < (1LL << 31) && encode_kc(&g.tmA, A, K, M, lda, sh.bm) &&
                       encode_kc(&g.tmB, B, K, N, ldb, sh.bn);
  if (use_sk) {
    dim3 grid((unsigned)gx, 1, 1);
    cudaError_t e;
    if (use_tma) e = launch_tma(cfg, st, g, grid);
    else if (akc && bkc) e = launch_layout<true, true>(cfg, st, g, grid);
    else if (akc && !bkc) e = launch_layout<true, false>(cfg, st, g, grid);
    else if (!akc && bkc) e = launch_layout<false, true>(cfg, st, g, grid);
    else e = launch_layout<false, false>(cfg, st, g, grid);
    c.launches += 1;
    c.flops += 2 * M * N * K;
    return e;
  }
  dim3 grid((unsigned)gx, (unsigned)gy, (unsigned)g.splits);
  cudaError_t e;
  if (use_tma) e = launch_tma(cfg, st, g, grid);
  else if (akc && bkc) e = launch_layout<true, true>(cfg, st, g, grid);
  else if (akc && !bkc) e = launch_layout<true, false>(cfg, st, g, grid);
  else if (!akc && bkc) e = launch_layout<false, true>(cfg, st, g, grid);
  else e = launch_layout<false, false>(cfg, st, g, grid);
  if (e != cudaSuccess) return e;
  c.launches += 1;
  c.flops += 2 * M * N * std::max<int64_t>(K, 0);
  if (g.splits > 1 && !pout) {
    const int64_t total = M * N;
    unsigned blocks = (unsigned)std::min<int64_t>((total + 255) / 256, 4096);
    gemm_splitk_reduce<<<blocks, 256, 0, st>>>(c.partial, g.splits, M, N, alpha, beta, C, ldc);
    c.launches += 1;
    e = cudaGetLastError();
  }
  return e;
}

}  // namespace ffb
