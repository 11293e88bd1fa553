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
//
// TMA variant (LOAD_TMA, both operands k-contiguous: the sketch B = Omega A and
// the WT products Y^T A): one elected thread issues cp.async.bulk.tensor 2-D
// loads of the (rows x 16) k-tiles into 128B-swizzled shared memory, completion
// is tracked by one mbarrier per stage (expect_tx), and edges are zero-filled by
// the TMA unit.  The 16-byte chunk c of tile row r sits at chunk c ^ (r & 7);
// DMMA fragment rows are taken in the order 0,2,4,6 | 1,3,5,7 within each 8-row
// group so that every half-warp's 16 doubles land on 16 distinct bank pairs.
#pragma once
#include <cuda.h>

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
  // stream-K: >0 => persistent grid, CTA b owns iterations [b*sk_per, (b+1)*sk_per)
  // of the linearised (tile, k-tile) space; every segment goes to
  // partial[(b*sk_maxseg + local)][BM*BN] and a fixup kernel sums them in order.
  int64_t sk_per;
  int sk_maxseg;
  int sk_tiles_n;    // tiles along N (tile = ty * sk_tiles_n + tx)
  int sk_lock;       // 1: the sk_tiles_n CTAs b*tn .. b*tn + tn - 1 walk the SAME (row block, k) range, one
                     // N tile each, in lockstep: the big row operand is read from HBM once and hits L2
                     // for the other N tiles (0: one linear range over all tiles per CTA)
  int64_t sk_kiters; // k-tiles per tile
  unsigned* sk_cnt;  // per-tile arrival counters (zero; reset by the last arriver)
  CUtensorMap tmA;   // LOAD_TMA: A as (K inner, M rows), box (16, BM), 128B swizzle
  CUtensorMap tmB;   // LOAD_TMA: B as (K inner, N rows), box (16, BN), 128B swizzle
};

// ---- TMA / mbarrier helpers (sm_90+ PTX; sm_100a here)
FFB_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
FFB_DEV void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
FFB_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
FFB_DEV void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n" ::
          "r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
FFB_DEV void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
// fragment row q (0..7) -> row inside its 8-row group (bank-conflict-free order)
FFB_DEV int tma_perm(int q) { return 2 * (q & 3) + (q >> 2); }
// double index of element (r, k) of a 128B-swizzled (rows x 16) k-tile
FFB_DEV int tma_idx(int r, int k) { return r * 16 + ((((k >> 1) ^ (r & 7))) << 1) + (k & 1); }

template <int BM, int BK>
struct APad {
  static constexpr int kc = BK + ((4 - BK % 16) + 16) % 16;        // (BK+pad) % 16 == 4
  // (BM+pad) % 16 == 4: a 64-bit fragment load's half-warp (4 k-rows x 4 rows)
  // then hits 16 distinct bank pairs (8 mod 16 put k-rows 0 and 2 on one bank)
  static constexpr int mc = BM + ((4 - BM % 16) + 16) % 16;
};

template <int BM, int BN, int BK, int WM, int WN, bool A_KC, bool B_KC, int STAGES, bool TMA = false>
struct GemmCfg {
  static constexpr int kWarpsM = BM / WM, kWarpsN = BN / WN;
  static constexpr int kThreads = 32 * kWarpsM * kWarpsN;
  static constexpr int kTM = WM / 8, kTN = WN / 8;
  // TMA: dense 128B-swizzled (rows x 16) tiles, 1024-byte aligned stages
  static constexpr int kAStage = TMA ? (BM * 16 + 127) / 128 * 128
                                     : (A_KC ? BM * APad<BM, BK>::kc : BK * APad<BM, BK>::mc);
  static constexpr int kBStage = TMA ? (BN * 16 + 127) / 128 * 128
                                     : (B_KC ? BN * APad<BN, BK>::kc : BK * APad<BN, BK>::mc);
  static constexpr size_t kStages = (size_t)STAGES * (kAStage + kBStage);
  static constexpr size_t kCTile = (size_t)(BM + 1) * BN;   // epilogue staging
  static constexpr size_t kSmem = sizeof(double) * (kStages > kCTile ? kStages : kCTile) + (TMA ? 1024 : 0);
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
  bool all_live;     // every row of the tile is in range (interior tiles)
  int nbf[kPer];     // cp.async source bytes of a full k-tile (row tail zero-filled)

  FFB_DEV void init(const double* base, int64_t ld, int64_t r0, int64_t rows, int64_t k0, int tid) {
    all_live = r0 + R <= rows;
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
      nbf[u] = !live[u] ? 0 : (VEC2 ? ((KC || gr + 1 < rows) ? 16 : 8) : 8);
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
  // interior tile with a full k-tile: no per-unit bounds, no zero-fill sizes
  FFB_DEV void load_full(double* smem) {
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      if (kUnits % NT != 0 && u * NT + (int)threadIdx.x >= kUnits) continue;
      double* dst = smem + soff[u];
      if (VEC2)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(g[u]));
      else
        cp_async8(dst, g[u], true);
    }
  }
  // full k-tile of an edge tile: per-unit byte counts fixed at init
  FFB_DEV void load_kfull(double* smem) {
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      if (kUnits % NT != 0 && u * NT + (int)threadIdx.x >= kUnits) continue;
      double* dst = smem + soff[u];
      if (VEC2)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)),
                     "l"(nbf[u] ? g[u] : g[0]), "r"(nbf[u]));
      else
        cp_async8(dst, nbf[u] ? g[u] : g[0], nbf[u] != 0);
    }
  }
  FFB_DEV void advance(int64_t ld) {
#pragma unroll
    for (int u = 0; u < kPer; ++u) g[u] += KC ? BK : (int64_t)BK * ld;
  }
};

template <int BM, int BN, int BK, int WM, int WN, bool A_KC, bool B_KC, int STAGES, bool VEC2,
          bool SK, bool TMA = false>
__global__ void __launch_bounds__(GemmCfg<BM, BN, BK, WM, WN, A_KC, B_KC, STAGES, TMA>::kThreads)
    gemm_f64_kernel(const __grid_constant__ GemmArgs g) {
  using Cfg = GemmCfg<BM, BN, BK, WM, WN, A_KC, B_KC, STAGES, TMA>;
  static_assert(!TMA || (A_KC && B_KC && BK == 16), "TMA path: k-contiguous operands, 16-wide k-tiles");
  constexpr int NT = Cfg::kThreads;
  constexpr int ALD = A_KC ? APad<BM, BK>::kc : APad<BM, BK>::mc;
  constexpr int BLD = B_KC ? APad<BN, BK>::kc : APad<BN, BK>::mc;
  extern __shared__ __align__(16) double smem_raw[];
  double* smem = TMA ? reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023))
                     : smem_raw;
  double* As = smem;
  double* Bs = smem + STAGES * Cfg::kAStage;
  __shared__ __align__(8) uint64_t full_bar[TMA ? STAGES : 1];
  uint32_t phases = 0;   // TMA: parity bit per stage of the next wait
  if (TMA) {
    if (threadIdx.x == 0) {
      for (int s = 0; s < STAGES; ++s) mbar_init(&full_bar[s], 1);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
  }

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm0 = (warp / Cfg::kWarpsN) * WM, wn0 = (warp % Cfg::kWarpsN) * WN;
  // segment loop: classic grid = one segment; stream-K = this CTA's iteration range
  int64_t it = 0, it_end = 1;
  constexpr bool sk = SK;
  // stream-K range owner and (lockstep mode) this CTA's N tile
  const int64_t sk_rng = sk && g.sk_lock ? (int64_t)blockIdx.x / g.sk_tiles_n : (int64_t)blockIdx.x;
  const int sk_nt = sk && g.sk_lock ? (int)(blockIdx.x % g.sk_tiles_n) : 0;
  if (sk) {
    it = sk_rng * g.sk_per;
    it_end = it + g.sk_per;
    const int64_t total = g.sk_kiters * ((g.M + BM - 1) / BM) * (g.sk_lock ? 1 : g.sk_tiles_n);
    if (it_end > total) it_end = total;
  }
  int local_seg = 0;
  const int64_t first_tile = sk ? it / g.sk_kiters : 0;
  for (; it < it_end; ++local_seg) {
  int64_t i0, j0, kbeg, kend;
  int split;
  int64_t sk_tile = 0, sk_lin = 0;   // output tile (counter index), tile index in the range space
  bool sk_whole = false;
  if (sk) {
    const int64_t tile = it / g.sk_kiters;
    const int64_t kb = it - tile * g.sk_kiters;
    int64_t ke = g.sk_kiters;
    if (ke - kb > it_end - it) ke = kb + (it_end - it);
    if (g.sk_lock) {
      i0 = tile * BM;
      j0 = (int64_t)sk_nt * BN;
      sk_tile = tile * g.sk_tiles_n + sk_nt;
    } else {
      i0 = (tile / g.sk_tiles_n) * BM;
      j0 = (tile % g.sk_tiles_n) * BN;
      sk_tile = tile;
    }
    sk_lin = tile;
    kbeg = kb * BK;
    kend = ke * BK < g.K ? ke * BK : g.K;
    split = (int)(blockIdx.x * g.sk_maxseg + (tile - first_tile));
    sk_whole = (kb == 0 && ke == g.sk_kiters);
    it += ke - kb;
  } else {
    i0 = (int64_t)blockIdx.y * BM;
    j0 = (int64_t)blockIdx.x * BN;
    split = blockIdx.z;
    kbeg = (int64_t)split * g.k_per;
    kend = min(g.K, kbeg + g.k_per);
    it = it_end;
  }
  const int nk = kbeg < kend ? (int)((kend - kbeg + BK - 1) / BK) : 0;
  if (TMA) fence_proxy_async_smem();   // epilogue's generic smem writes before the next TMA fills
  __syncthreads();   // previous segment's smem reads done before refilling

  TileLoader<BM, BK, A_KC, VEC2, NT> la;
  TileLoader<BN, BK, B_KC, VEC2, NT> lb;
  if (!TMA) {
    la.init(g.A, g.lda, i0, g.M, kbeg, tid);
    lb.init(g.B, g.ldb, j0, g.N, kbeg, tid);
  }

  double acc[Cfg::kTM][Cfg::kTN][2];
#pragma unroll
  for (int a = 0; a < Cfg::kTM; ++a)
#pragma unroll
    for (int b = 0; b < Cfg::kTN; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  int fetched = 0;
  auto fetch = [&](int stage) {
    if constexpr (TMA) {
      if (tid == 0) {
        const int k0 = (int)(kbeg + (int64_t)fetched * BK);
        mbar_expect_tx(&full_bar[stage], (uint32_t)((BM + BN) * BK * sizeof(double)));
        tma_load_2d(As + stage * Cfg::kAStage, &g.tmA, &full_bar[stage], k0, (int)i0);
        tma_load_2d(Bs + stage * Cfg::kBStage, &g.tmB, &full_bar[stage], k0, (int)j0);
      }
      ++fetched;
      return;
    }
    const int64_t k0 = kbeg + (int64_t)fetched * BK;
    const int64_t krem = kend - k0;
    const int kvalid = krem < BK ? (int)krem : BK;
    if (kvalid == BK) {
      if (la.all_live) la.load_full(As + stage * Cfg::kAStage);
      else la.load_kfull(As + stage * Cfg::kAStage);
      if (lb.all_live) lb.load_full(Bs + stage * Cfg::kBStage);
      else lb.load_kfull(Bs + stage * Cfg::kBStage);
    } else {
      la.load(As + stage * Cfg::kAStage, kvalid, i0, g.M, g.lda);
      lb.load(Bs + stage * Cfg::kBStage, kvalid, j0, g.N, g.ldb);
    }
    la.advance(g.lda);
    lb.advance(g.ldb);
    ++fetched;
  };

#pragma unroll
  for (int st = 0; st < STAGES - 1; ++st) {
    if (st < nk) fetch(st);
    if (!TMA) cp_async_commit();
  }

  const int fr = lane >> 2, fk = lane & 3;
  const int frp = TMA ? tma_perm(fr) : fr;   // fragment row -> tile row inside the 8-row group
  // TMA: element (r, 4q + fk) of a swizzled tile sits at r*16 + (fk & 1) + (4q ^ c0)
  // with c0 = ((fk >> 1) ^ (r & 7)) << 1 (r & 7 = frp for every fragment row)
  const int tma_c0 = ((fk >> 1) ^ frp) << 1;
  const int tma_a0 = (wm0 + frp) * 16 + (fk & 1);
  const int tma_b0 = (wn0 + frp) * 16 + (fk & 1);
  for (int kt = 0; kt < nk; ++kt) {
    if (!TMA) cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int pf = kt + STAGES - 1;
      if (pf < nk) fetch(pf % STAGES);
      if (!TMA) cp_async_commit();
    }
    if (TMA) {
      const int s_ = kt % STAGES;
      mbar_wait(&full_bar[s_], (phases >> s_) & 1u);
      phases ^= 1u << s_;
    }
    const double* as = As + (kt % STAGES) * Cfg::kAStage;
    const double* bs = Bs + (kt % STAGES) * Cfg::kBStage;
    // fragments double-buffered across the k4 steps: the loads for step k4 + 4
    // are issued before the DMMAs of step k4, so no DMMA waits on a fresh LDS and
    // no LDS overwrites a register an in-flight DMMA still reads
    double af[2][Cfg::kTM], bf[2][Cfg::kTN];
    auto load_frag = [&](int k4, double (&a_)[Cfg::kTM], double (&b_)[Cfg::kTN]) {
      if constexpr (TMA) {
        const int x = k4 ^ tma_c0;   // k4 = 4q is a compile-time constant
        const double* pa = as + tma_a0 + x;
        const double* pb = bs + tma_b0 + x;
#pragma unroll
        for (int a = 0; a < Cfg::kTM; ++a) a_[a] = pa[a * 128];   // 8 rows x 16 doubles per fragment
#pragma unroll
        for (int b = 0; b < Cfg::kTN; ++b) b_[b] = pb[b * 128];
        return;
      }
#pragma unroll
      for (int a = 0; a < Cfg::kTM; ++a) {
        const int r = wm0 + a * 8 + frp, kk = k4 + fk;
        a_[a] = A_KC ? as[r * ALD + kk] : as[kk * ALD + r];
      }
#pragma unroll
      for (int b = 0; b < Cfg::kTN; ++b) {
        const int c = wn0 + b * 8 + frp, kk = k4 + fk;
        b_[b] = B_KC ? bs[c * BLD + kk] : bs[kk * BLD + c];
      }
    };
    load_frag(0, af[0], bf[0]);
#pragma unroll
    for (int k4 = 0; k4 < BK; k4 += 4) {
      const int cur = (k4 >> 2) & 1;
      if (k4 + 4 < BK) load_frag(k4 + 4, af[cur ^ 1], bf[cur ^ 1]);
#pragma unroll
      for (int a = 0; a < Cfg::kTM; ++a)
#pragma unroll
        for (int b = 0; b < Cfg::kTN; ++b)
          dmma_884(acc[a][b][0], acc[a][b][1], af[cur][a], bf[cur][b]);
    }
  }
  if (!TMA) cp_async_wait<0>();

  // Epilogue: stage the accumulator tile in shared memory (column-major, ld
  // BM + 1), then one compact coalesced loop writes it out (C, a split-K slab
  // or a stream-K segment).  Keeps the kernel's code small (instruction cache)
  // and the global stores contiguous along M.
  constexpr int CLD = BM + 1;
  __syncthreads();
  double* Ct = smem;
#pragma unroll
  for (int a = 0; a < Cfg::kTM; ++a)
#pragma unroll
    for (int b = 0; b < Cfg::kTN; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int cq = TMA ? tma_perm(2 * fk + h) : 2 * fk + h;
        Ct[(wm0 + a * 8 + frp) + (wn0 + b * 8 + cq) * CLD] = acc[a][b][h];
      }
  __syncthreads();
  {
    // destination: 0 = C (alpha, beta), 1 = partial slab (raw)
    int mode;
    double* dst;
    int64_t ldd;
    if (sk) {
      mode = sk_whole ? 0 : 1;
      dst = sk_whole ? g.C + i0 + j0 * g.ldc : g.partial + (size_t)split * (BM * BN);
      ldd = sk_whole ? g.ldc : BM;
    } else if (g.splits == 1 && !g.force_partial) {
      mode = 0;
      dst = g.C + i0 + j0 * g.ldc;
      ldd = g.ldc;
    } else {
      mode = 1;
      dst = g.partial + (size_t)split * g.M * g.N + i0 + j0 * g.M;
      ldd = g.M;
    }
    const int rmax = g.M - i0 < BM ? (int)(g.M - i0) : BM;
    const int cmax = g.N - j0 < BN ? (int)(g.N - j0) : BN;
    const double alpha = g.alpha, beta = g.beta;
    const bool rd = mode == 0 && beta != 0.0;
    // C reads are issued 8 at a time before their uses (no serial L2 round trips)
    constexpr int EPT = (BM * BN + NT - 1) / NT;
    constexpr int G8 = 8;
#pragma unroll 1
    for (int q0 = 0; q0 < EPT; q0 += G8) {
      double cv[G8];
#pragma unroll
      for (int u = 0; u < G8; ++u) {
        const int e = tid + (q0 + u) * NT;
        const int r = e % BM, c = e / BM;
        cv[u] = (rd && q0 + u < EPT && e < BM * BN && r < rmax && c < cmax) ? dst[r + (int64_t)c * ldd] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < G8; ++u) {
        const int e = tid + (q0 + u) * NT;
        const int r = e % BM, c = e / BM;
        if (q0 + u >= EPT || e >= BM * BN || r >= rmax || c >= cmax) continue;
        const double v = Ct[r + c * CLD];
        dst[r + (int64_t)c * ldd] = mode == 1 ? v : (rd ? alpha * v + beta * cv[u] : alpha * v);
      }
    }
  }
  if (sk && !sk_whole) {
    // last CTA to finish this tile reduces every segment in CTA order -> C
    __shared__ int s_last;
    __syncthreads();
    const int64_t t0 = sk_lin * g.sk_kiters, t1 = t0 + g.sk_kiters - 1;
    const int64_t b0 = t0 / g.sk_per, b1 = t1 / g.sk_per;
    if (tid == 0) {
      __threadfence();
      const unsigned old = atomicAdd(g.sk_cnt + sk_tile, 1u);
      s_last = (old == (unsigned)(b1 - b0));
    }
    __syncthreads();
    if (s_last) {
      __threadfence();
      __shared__ const double* segp[16];
      if (tid <= (int)(b1 - b0) && tid < 16) {
        const int64_t bq = b0 + tid;   // range owner; its CTA for this N tile in lockstep mode
        const int64_t ft = (bq * g.sk_per) / g.sk_kiters;
        const int64_t blk = g.sk_lock ? bq * g.sk_tiles_n + sk_nt : bq;
        segp[tid] = g.partial + (size_t)(blk * g.sk_maxseg + (sk_lin - ft)) * (BM * BN);
      }
      __syncthreads();
      const int ns = (int)(b1 - b0 + 1);
      // 8 elements per thread per pass: their segment loads are in flight together
      // (each element still sums its segments in ascending order)
      constexpr int EPT = (BM * BN + NT - 1) / NT;
      for (int e0 = 0; e0 < EPT; e0 += 8) {
        double sum[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) sum[u] = 0.0;
        for (int q = 0; q < ns; ++q) {
          double v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int e = tid + (e0 + u) * NT;
            v[u] = (e0 + u < EPT && e < BM * BN) ? __ldcg(segp[q] + e) : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) sum[u] += v[u];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int e = tid + (e0 + u) * NT;
          if (e0 + u >= EPT || e >= BM * BN) continue;
          const int r = e % BM, c = e / BM;
          const int64_t gi = i0 + r, gj = j0 + c;
          if (gi >= g.M || gj >= g.N) continue;
          double* cp = g.C + gi + gj * g.ldc;
          const double v = g.alpha * sum[u];
          *cp = g.beta == 0.0 ? v : v + g.beta * (*cp);
        }
      }
      if (tid == 0) g.sk_cnt[sk_tile] = 0u;
    }
  }
  }  // segment loop
}

// Fixed-order reduction of split-K partials into C.  The partial loads are
// issued 8 at a time (independent, in flight together) and summed in split
// order: a serial chain of L2 round trips made this kernel ~10 us for the
// small-output, long-K products of the panel updates.
__global__ void gemm_splitk_reduce(const double* __restrict__ part, int splits, int64_t M, int64_t N,
                                   double alpha, double beta, double* C, int64_t ldc) {
  const int64_t total = M * N;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    int q = 0;
    for (; q + 8 <= splits; q += 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldcg(part + (size_t)(q + u) * total + t);
#pragma unroll
      for (int u = 0; u < 8; ++u) s += v[u];
    }
    for (; q < splits; ++q) s += __ldcg(part + (size_t)q * total + t);
    const int64_t i = t % M, j = t / M;
    double* cp = C + i + j * ldc;
    const double v = alpha * s;
    *cp = beta == 0.0 ? v : v + beta * (*cp);
  }
}

}  // namespace ffb
