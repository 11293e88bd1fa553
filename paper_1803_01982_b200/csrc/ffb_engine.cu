// Orchestrator and C ABI of the B200 Flip-Flop SRQR engine.
//
// One call = one factorization, enqueued on the caller's stream with no host
// synchronisation until the end: TRQRCP (sketch GEMM, per-block cooperative
// pivot kernel, CholeskyQR3 + Householder-reconstruction panels, compact-WY
// GEMMs), SRQR (extension, g2 estimate, pack) and — speculatively, assuming
// the first g2 test certifies — the flip-flop tail (partial LQ, A*Qhat,
// small SVD, back-mapping).  A single sync at the end reads the certificate;
// only if a swap is needed (g2 > g, rare: 0 swaps on every BASELINE config)
// does the host drive the reference's swap loop and redo the tail.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <atomic>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <unordered_map>
#include <vector>

#include "../../include/ffb200.h"
#include "ffb_gemm.h"
#include "ffb_jacobi.cuh"
#include "ffb_kernels.cuh"
#include "ffb_panel.cuh"

using namespace ffb;

// A captured launch sequence (ffb_run's core) and the bookkeeping it adds.
struct GraphEnt {
  cudaGraphExec_t exec = nullptr;
  int64_t launches = 0, glaunches = 0, flops = 0;
  uint64_t stamp = 0;
};

struct ffb_ctx {
  int device = 0;
  int sms = 148;
  int max_coop_blocks_smem = 0;
  std::string err;
  std::mutex err_mu;               // problems of a batch may fail concurrently
  double* pinned = nullptr;        // host staging for g2 Gaussians
  size_t pinned_cap = 0;
  SrqrScalars* sc_host = nullptr;  // pinned
  std::mutex gmu;                  // graph cache (several host threads per context)
  std::unordered_map<std::string, GraphEnt> graphs;
  std::vector<cudaGraphExec_t> retired;
  uint64_t gstamp = 0;
};

namespace {

// Host staging is per calling thread, so independent problems can be driven from
// several host threads / CUDA streams on one context (batch.run_streams).
struct HostStage {
  double* pinned = nullptr;        // g2 Gaussians
  size_t cap = 0;
  cudaStream_t capture[64] = {};   // per device: private stream the graph capture records on
  SrqrScalars* sc = nullptr;       // certificate scalars read back after the pipeline
  unsigned char* small = nullptr;  // 256 B: small read-backs (status words, sweep counts)
  ~HostStage() {
    if (pinned) cudaFreeHost(pinned);
    if (sc) cudaFreeHost(sc);
    if (small) cudaFreeHost(small);
  }
};
thread_local HostStage t_host;

// SMs one problem may spread its cooperative kernels over (0 = the whole
// device): batch drivers with S problems in flight give each ~SMs / S, so the
// problems' grid-synchronised kernels are co-resident instead of queueing.
thread_local int t_sm_budget = 0;

int effective_sms(const ffb_ctx* ctx) {
  const int all = ctx ? ctx->sms : 148;
  return t_sm_budget > 0 ? std::min(t_sm_budget, all) : all;
}

// small stream-ordered read-back (<= 256 B).  An SM kernel writes the pinned
// staging word (UVA) instead of a D2H memcpy: the copy engines' queues, where
// another stream's large transfer may be in flight, stay off the critical path.
inline cudaError_t d2h(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (!t_host.small) {
    cudaError_t e = cudaMallocHost(&t_host.small, 256);
    if (e != cudaSuccess) return e;
  }
  cudaError_t e = launch_copy_bytes(st, src, t_host.small, bytes);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e == cudaSuccess) memcpy(dst, t_host.small, bytes);
  return e;
}

// device-to-device copies on the SMs (see d2h)
inline cudaError_t d2d(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  return launch_copy_bytes(st, src, dst, bytes);
}

constexpr int kPanelW = 64;

// column width of the Householder panels hh_qr factors in one fused kernel
// (<= kPanelW; FFB_PANEL_W tunes it): narrower panels shorten the serial
// Cholesky / sign-LU chains at the cost of more trailing-update GEMMs
int panel_step() {
  static int w = -1;
  if (w < 0) {
    const char* e = getenv("FFB_PANEL_W");
    w = e ? std::max(8, std::min(kPanelW, atoi(e))) : kPanelW;
  }
  return w;
}
constexpr size_t kAlign = 256;

struct Bump {
  char* base;
  size_t off = 0;
  size_t cap;
  bool ok = true;
  template <typename T>
  T* take(size_t count) {
    off = (off + kAlign - 1) / kAlign * kAlign;
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += std::max<size_t>(count, 1) * sizeof(T);
    if (off > cap) ok = false;
    return p;
  }
};

struct Dims {
  int64_t m, n, k, l, b, p, s, d;
  double g;
  uint64_t seed;
  int mode;
};

struct Work {
  // TRQRCP
  double *B, *colsq, *Y, *T, *WT, *R, *Q;
  int64_t *arr, *pos;
  double *P, *Xa, *Xb, *G1, *WTg, *S1, *S2, *Racc, *Gm, *ppart, *Rinv, *Ut, *Dv, *Rb, *Bp, *Z;
  uint32_t* pbar;
  double *hhW, *hhW2;
  // pivots
  unsigned long long* prec;
  double *slotdata, *pwork, *gap;
  uint32_t* flags;
  int64_t* hist;
  int G, cpc;
  bool piv_smem;
  size_t piv_smem_bytes;
  // SRQR
  double *r, *rinit, *u, *ct, *part, *rot, *g2om, *g2z, *g2R, *cpart;
  uint32_t* g2flag;
  SrqrScalars* sc;
  uint32_t* status;
  // flip-flop
  double *X, *Yl, *Tl, *Rl, *TYt, *Qh, *Yh, *tmp, *Yt, *Tt, *Rt, *Us, *jwork, *Vo, *sig, *W1, *W2;
  double* joff;
  uint32_t* jbar;
  int *jsweeps, *jorder;
  double* gpart;
  size_t gpart_cap;
  unsigned* skcnt;
};

int64_t max_i(int64_t a, int64_t b) { return a > b ? a : b; }

// Pivot-kernel geometry: G CTAs (<= #SMs, ~64 columns each), columns in
// shared memory when they fit.
void pivot_geometry(const ffb_ctx* ctx, int64_t n, int64_t s, Work& w) {
  int gmax = std::min(effective_sms(ctx), 160);   // kPivMaxK * 32
  if (const char* ev = getenv("FFB_PIV_G")) gmax = std::max(1, std::min(gmax, atoi(ev)));
  // 64 columns per CTA (the register-resident maximum) when the grid allows:
  // fewer CTAs shorten the per-step all-CTA exchange
  int G = (int)std::min<int64_t>(gmax, std::max<int64_t>(1, (n + 63) / 64));
  int cpc = (int)((n + G - 1) / G);
  const size_t smem_all = pivots_smem_bytes((int)s, cpc, true);
  w.piv_smem = smem_all <= 200 * 1024;
  w.G = G;
  w.cpc = cpc;
  w.piv_smem_bytes = pivots_smem_bytes((int)s, cpc, w.piv_smem);
}

constexpr int kMaxSweeps = 30;   // LAPACK dgesvj's sweep cap

size_t carve(const ffb_ctx* ctx, const Dims& D, void* base, size_t cap, Work& w) {
  Bump b{static_cast<char*>(base), 0, cap};
  const int64_t m = D.m, n = D.n, l = D.l, s = D.s, bmax = std::min<int64_t>(D.b, l);
  const int64_t L1 = l + 1;
  const int64_t mn = max_i(m, n);
  w.B = b.take<double>(s * n);
  w.colsq = b.take<double>(n);
  w.cpart = b.take<double>(colsq_rm_part_doubles(n));   // row-major A: column-norm partials
  w.arr = b.take<int64_t>(n);
  w.pos = b.take<int64_t>(n);
  w.Y = b.take<double>(m * l);
  w.T = b.take<double>(l * l);
  w.WT = b.take<double>(l * n);
  w.R = b.take<double>(L1 * n);
  w.Q = b.take<double>(m * L1);
  w.P = b.take<double>(m * bmax);
  w.Xa = b.take<double>(mn * kPanelW);
  w.Xb = b.take<double>(mn * kPanelW);
  w.G1 = b.take<double>(bmax * n);
  w.WTg = b.take<double>(l * bmax);
  w.S1 = b.take<double>(max_i(l, 1) * max_i(bmax, kPanelW));
  w.S2 = b.take<double>(max_i(l, 1) * max_i(bmax, kPanelW));
  w.Racc = b.take<double>(kPanelW * kPanelW);
  w.Gm = b.take<double>(kPanelW * kPanelW);
  w.ppart = b.take<double>((size_t)(ctx ? ctx->sms : 160) * kPanelW * kPanelW);
  w.pbar = b.take<uint32_t>(4);
  w.Rinv = b.take<double>(max_i(kPanelW * kPanelW, bmax * bmax));
  w.Ut = b.take<double>(kPanelW * kPanelW);
  w.Dv = b.take<double>(kPanelW);
  w.Rb = b.take<double>(bmax * bmax);
  w.Bp = b.take<double>(s * bmax);
  w.Z = b.take<double>(s * bmax);
  w.hhW = b.take<double>(kPanelW * max_i(l, 1));
  w.hhW2 = b.take<double>(kPanelW * max_i(l, 1));
  pivot_geometry(ctx, n, s, w);
  // sized for any grid the SM budget may pick (G <= 160, G * cpc < n + G)
  w.prec = b.take<unsigned long long>(2 * (size_t)160 * pivots_recw((int)s));
  w.hist = b.take<int64_t>(max_i(D.b, 1));
  w.gap = b.take<double>(max_i(l, 1));
  w.pwork = w.piv_smem ? nullptr : b.take<double>((size_t)(n + 160) * pivots_stride((int)s));
  w.r = b.take<double>(n);
  w.rinit = b.take<double>(n);
  w.u = b.take<double>(m);
  w.ct = b.take<double>(L1);
  w.part = b.take<double>(max_i(4096, (m + 255) / 256 + 1));
  w.rot = b.take<double>(4 * L1 + 8);
  w.g2om = b.take<double>(D.d * L1);
  w.g2z = b.take<double>(D.d * L1);
  w.g2R = L1 > 1024 ? b.take<double>(L1 * L1) : nullptr;   // explicit Rtilde, blocked g2 solve
  w.g2flag = b.take<uint32_t>(1);
  w.sc = b.take<SrqrScalars>(1);
  w.status = b.take<uint32_t>(1);
  w.TYt = b.take<double>(l * l);
  if (D.mode == FFB_MODE_FLIPFLOP) {
    w.X = b.take<double>(n * l);
    w.Yl = b.take<double>(n * l);
    w.Tl = b.take<double>(l * l);
    w.Rl = b.take<double>(l * l);
    w.Qh = b.take<double>(n * l);
    w.Yh = b.take<double>(n * l);
    w.tmp = b.take<double>(m * l);
    w.Yt = b.take<double>(m * l);
    w.Tt = b.take<double>(l * l);
    w.Rt = b.take<double>(l * l);
    w.Us = b.take<double>(l * l);
    w.jwork = b.take<double>(jacobi_work_doubles((int)l, kMaxSweeps));
    w.Vo = b.take<double>(l * l);
    w.sig = b.take<double>(l);
    w.W1 = b.take<double>(l * D.k);
    w.W2 = b.take<double>(l * D.k);
    w.joff = b.take<double>(kMaxSweeps);
    w.jbar = b.take<uint32_t>(4);
    w.jsweeps = b.take<int>(4);
    w.jorder = b.take<int>(l);
  }
  // split-K scratch: the rest, at least 4 Mi doubles
  w.gpart_cap = std::max<size_t>(16u << 20, (size_t)64 * kPanelW * kPanelW);
  w.gpart = b.take<double>(w.gpart_cap);
  w.skcnt = b.take<unsigned>(65536);
  return b.off + kAlign;
}

// Workspace of the randomized subspace-iteration SVD (ffb_rsisvd): the rank-r
// working matrices plus the same panel / Jacobi / GEMM scratch as the flip-flop.
size_t carve_rsisvd(const ffb_ctx* ctx, int64_t m, int64_t n, int64_t k, int64_t r, void* base,
                    size_t cap, Work& w) {
  Bump b{static_cast<char*>(base), 0, cap};
  const int64_t mn = max_i(m, n);
  w.tmp = b.take<double>(m * r);      // A Omega, A Q_z (factored in place)
  w.Yt = b.take<double>(m * r);       // reflectors of the m x r QRs
  w.Tt = b.take<double>(r * r);
  w.Rt = b.take<double>(r * r);
  w.Q = b.take<double>(m * r);        // explicit Q (m x r)
  w.X = b.take<double>(n * r);        // A^T Q (factored in place)
  w.Yl = b.take<double>(n * r);       // reflectors of the n x r QRs
  w.Tl = b.take<double>(r * r);
  w.Rl = b.take<double>(r * r);
  w.Qh = b.take<double>(n * r);       // explicit Q_z (n x r)
  w.TYt = b.take<double>(r * r);
  w.Xa = b.take<double>(mn * kPanelW);
  w.Xb = b.take<double>(mn * kPanelW);
  w.S1 = b.take<double>(r * kPanelW);
  w.S2 = b.take<double>(r * kPanelW);
  w.Gm = b.take<double>(kPanelW * kPanelW);
  w.ppart = b.take<double>((size_t)(ctx ? ctx->sms : 160) * kPanelW * kPanelW);
  w.pbar = b.take<uint32_t>(4);
  w.hhW = b.take<double>(kPanelW * r);
  w.hhW2 = b.take<double>(kPanelW * r);
  w.status = b.take<uint32_t>(1);
  w.Us = b.take<double>(r * r);
  w.Vo = b.take<double>(r * r);
  w.sig = b.take<double>(r);
  w.jwork = b.take<double>(jacobi_work_doubles((int)r, kMaxSweeps));
  w.W1 = b.take<double>(r * k);
  w.W2 = b.take<double>(r * k);
  w.joff = b.take<double>(kMaxSweeps);
  w.jbar = b.take<uint32_t>(4);
  w.jsweeps = b.take<int>(4);
  w.jorder = b.take<int>(r);
  w.gpart_cap = std::max<size_t>(16u << 20, (size_t)64 * kPanelW * kPanelW);
  w.gpart = b.take<double>(w.gpart_cap);
  w.skcnt = b.take<unsigned>(65536);
  return b.off + kAlign;
}

// The input matrix A (m x n) in the caller's storage: column-major
// (A(i, j) = p[i + j*ld]) or row-major (p[i*ld + j], FFB_LAYOUT_ROW).
struct AView {
  const double* p;
  int64_t ld;
  bool row;
  const double* rows_from(int64_t i0) const { return row ? p + i0 * ld : p + i0; }
  int64_t rs() const { return row ? ld : 1; }   // stride between rows
  int64_t cs() const { return row ? 1 : ld; }   // stride between columns
  bool kc_as_b() const { return !row; }          // as GEMM B operand with k = row index
  bool kc_as_a() const { return row; }           // as GEMM A operand with k = column index
};

struct Eng {
  ffb_ctx* ctx;
  int sms = 148;                   // SM budget of this problem (effective_sms)
  cudaStream_t st;
  Dims D;
  Work w;
  GemmCtx gc;
  int64_t launches = 0;
  cudaError_t cerr = cudaSuccess;

  bool ok(cudaError_t e) {
    if (e != cudaSuccess && cerr == cudaSuccess) cerr = e;
    ++launches;
    return e == cudaSuccess;
  }
  // stream memsets: checked like launches but not counted as kernels
  bool okm(cudaError_t e) {
    if (e != cudaSuccess && cerr == cudaSuccess) cerr = e;
    return e == cudaSuccess;
  }
  void gemm(int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda, bool akc,
            const double* B, int64_t ldb, bool bkc, double beta, double* C, int64_t ldc) {
    if (cerr != cudaSuccess) return;
    cudaError_t e = gemm_f64(gc, st, M, N, K, alpha, A, lda, akc, B, ldb, bkc, beta, C, ldc);
    if (e != cudaSuccess) cerr = e;
  }
  // Gram G = X^T X (w x w, reduced in fixed order) of X (rows x w, ld ldx)
  void gram(const double* X, int64_t rows, int w_, int64_t ldx) {
    gemm(w_, w_, rows, 1.0, X, ldx, true, X, ldx, true, 0.0, w.Gm, w_);
  }
  void memset2d(double* p, int64_t ld, int64_t rows, int64_t cols) {
    if (rows <= 0 || cols <= 0) return;
    okm(cudaMemset2DAsync(p, ld * sizeof(double), 0, rows * sizeof(double), cols, st));
  }

  // g2 estimate (srqr.py:49-64): one-thread-per-row kernel for l + 1 <= 1024,
  // else blocked back substitution (diagonal blocks of 1024 + GEMM updates)
  void g2() {
    const int64_t l = D.l, L1 = l + 1;
    if (L1 <= 1024) {
      ok(launch_g2(st, w.R, L1, w.arr, l, w.g2om, (int)D.d, D.g, w.g2z, w.sc));
      return;
    }
    ok(launch_r_arranged(st, w.R, L1, w.arr, L1, L1, w.g2R, L1, L1));
    ok(launch_g2big_prep(st, w.g2R, L1, w.g2om, (int)D.d, w.g2z, w.sc, w.g2flag));
    constexpr int64_t kBlk = 1024;
    for (int64_t i1 = L1; i1 > 0; i1 -= kBlk) {
      const int64_t i0 = std::max<int64_t>(0, i1 - kBlk);
      ok(launch_g2big_diag(st, w.g2R, L1, i0, (int)(i1 - i0), w.g2z, (int)D.d));
      if (i0 > 0)
        gemm(i0, D.d, i1 - i0, -1.0, w.g2R + i0 * L1, L1, false, w.g2z + i0, L1, true, 1.0, w.g2z, L1);
    }
    ok(launch_g2big_finish(st, w.g2z, L1, (int)D.d, D.g, w.g2flag, w.sc));
  }

  // Rinv (ld ldo) = Rb^{-1} for an upper-triangular bb x bb block (ld ldr): one
  // tile kernel for bb <= 64, else recursively in the 2 x 2 block form
  // [A B; 0 C]^{-1} = [A^-1, -A^-1 B C^-1; 0, C^-1] (two half inverses + 2 GEMMs)
  void tri_inverse(const double* Rb, int64_t ldr, int64_t bb, double* Rinv, int64_t ldo) {
    if (bb <= kPanelW) {
      ok(launch_triinv_upper(st, Rb, ldr, (int)bb, Rinv, ldo, w.status));
      return;
    }
    const int64_t h = std::max<int64_t>(kPanelW, (bb / 2 + kPanelW - 1) / kPanelW * kPanelW);
    const int64_t t = bb - h;
    tri_inverse(Rb, ldr, h, Rinv, ldo);
    tri_inverse(Rb + h + h * ldr, ldr, t, Rinv + h + h * ldo, ldo);
    memset2d(Rinv + h, ldo, t, h);
    // S2 (h x t) = B C^-1 ; Rinv12 = -A^-1 S2
    gemm(h, t, t, 1.0, Rb + h * ldr, ldr, false, Rinv + h + h * ldo, ldo, true, 0.0, w.S2, h);
    gemm(h, t, h, -1.0, Rinv, ldo, false, w.S2, h, true, 0.0, Rinv + h * ldo, ldo);
  }

  // Householder panel (Mp x wb, wb <= 64): one fused cooperative kernel
  // (shifted CholeskyQR3 + Householder reconstruction, ffb_panel.cu).
  void recon(const double* Xp, int64_t Mp, int wb, int64_t ldx, double* Yp, int64_t ldy,
             double* Tp, int64_t ldt, double* Rp, int64_t ldr) {
    if (cerr != cudaSuccess) return;
    ok(launch_panel_qr(st, sms, Xp, ldx, Mp, wb, Yp, ldy, Tp, ldt, Rp, ldr, w.Xa, w.Xb,
                       w.ppart, w.Gm, w.pbar, w.status));
    gc.flops += 3 * 4 * Mp * (int64_t)wb * wb + 2 * Mp * (int64_t)wb * wb;
  }

  // Blocked Householder QR of X (Mx x Nx, ld ldx), panels of <= 64 columns.
  // Y (ld ldy), T (ld ldt), R (ld ldr): R gets the diagonal blocks, and the full
  // upper triangle when full_r.  X is overwritten by the trailing updates.
  void hh_qr(double* X, int64_t Mx, int64_t Nx, int64_t ldx, double* Y, int64_t ldy, double* T,
             int64_t ldt, double* R, int64_t ldr, bool full_r) {
    memset2d(Y, ldy, Mx, Nx);
    memset2d(T, ldt, Nx, Nx);
    memset2d(R, ldr, Nx, Nx);
    const int pw = panel_step();
    for (int64_t c0 = 0; c0 < Nx; c0 += pw) {
      const int64_t c1 = std::min<int64_t>(Nx, c0 + pw);
      const int wb = (int)(c1 - c0);
      const int64_t Mp = Mx - c0;
      double* Yp = Y + c0 + c0 * ldy;
      double* Tp = T + c0 + c0 * ldt;
      recon(X + c0 + c0 * ldx, Mp, wb, ldx, Yp, ldy, Tp, ldt, R + c0 + c0 * ldr, ldr);
      if (c1 < Nx) {
        const int64_t Nt = Nx - c1;
        gemm(wb, Nt, Mp, 1.0, Yp, ldy, true, X + c0 + c1 * ldx, ldx, true, 0.0, w.hhW, wb);
        gemm(wb, Nt, wb, 1.0, Tp, ldt, true, w.hhW, wb, true, 0.0, w.hhW2, wb);
        gemm(Mp, Nt, wb, -1.0, Yp, ldy, false, w.hhW2, wb, true, 1.0, X + c0 + c1 * ldx, ldx);
        if (full_r) ok(launch_copy_rows(st, X + c0 + c1 * ldx, ldx, wb, Nt, R + c0 + c1 * ldr, ldr));
      }
      if (c0 > 0) {
        // T12 = -T11 (Y1^T Y2) T22 ; Y2 is zero above row c0
        gemm(c0, wb, Mx - c0, 1.0, Y + c0, ldy, true, Yp, ldy, true, 0.0, w.S1, c0);
        gemm(c0, wb, wb, 1.0, w.S1, c0, false, Tp, ldt, true, 0.0, w.S2, c0);
        gemm(c0, wb, c0, -1.0, T, ldt, false, w.S2, c0, true, 0.0, T + c0 * ldt, ldt);
      }
    }
  }
};


// Q[:, :Nx] = (I - Y T Y_top^T)[:, :Nx] explicitly (Mx x Nx, ld ldq) from a hh_qr
// factorization: LAPACK dorgqr's thin Q, as numpy.linalg.qr returns it.
void explicit_q(Eng& e, const double* Y, int64_t ldy, const double* T, int64_t ldt, int64_t Mx,
                int64_t Nx, double* Q, int64_t ldq) {
  e.gemm(Nx, Nx, Nx, 1.0, T, ldt, false, Y, ldy, false, 0.0, e.w.TYt, Nx);
  e.gemm(Mx, Nx, Nx, -1.0, Y, ldy, false, e.w.TYt, Nx, true, 0.0, Q, ldq);
  e.ok(launch_add_identity(e.st, Q, ldq, Mx, Nx, 1.0));
}

// The message of the last failing call made on this thread (errno-like):
// problems of a batch may fail concurrently on other threads, so a shared
// string could be reassigned while a caller reads it.
thread_local std::string t_err;

int fail(ffb_ctx* ctx, int code, const std::string& msg) {
  t_err = msg;
  if (ctx) {
    std::lock_guard<std::mutex> g(ctx->err_mu);
    ctx->err = msg;
  }
  return code;
}

// Makes `dev` current for the duration of an entry point and restores the
// caller's current device afterwards.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

int cuda_fail(ffb_ctx* ctx, cudaError_t e, const char* where) {
  return fail(ctx, FFB_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

// ---- concurrent-call tracking for graph capture.  A capture must not overlap
// another thread's launches: with lazy module loading, a kernel loaded for the
// first time during another thread's capture fails with "operation not
// permitted when stream is capturing" (seen with 8 batch threads).  So a
// capture only starts when this is the only call in flight, new calls wait
// until it ends, and once calls have overlapped the process stops capturing
// (cached graphs still replay).
std::atomic<int> g_inflight{0};
std::atomic<bool> g_capturing{false};
std::atomic<bool> g_ever_concurrent{false};
std::mutex g_cap_mu;
std::condition_variable g_cap_cv;

struct CallGuard {
  CallGuard() {
    if (g_inflight.fetch_add(1) + 1 > 1) g_ever_concurrent.store(true);
    if (g_capturing.load()) {
      std::unique_lock<std::mutex> lk(g_cap_mu);
      g_cap_cv.wait(lk, [] { return !g_capturing.load(); });
    }
  }
  ~CallGuard() { g_inflight.fetch_sub(1); }
};

bool begin_exclusive_capture() {
  if (g_ever_concurrent.load()) return false;
  g_capturing.store(true);
  if (g_inflight.load() != 1) {
    g_capturing.store(false);
    std::lock_guard<std::mutex> lk(g_cap_mu);
    g_cap_cv.notify_all();
    return false;
  }
  return true;
}

void end_exclusive_capture() {
  g_capturing.store(false);
  std::lock_guard<std::mutex> lk(g_cap_mu);
  g_cap_cv.notify_all();
}

// ---- CUDA graph cache of ffb_run's core (FFB_GRAPHS=0 disables it)
constexpr size_t kMaxGraphs = 256;

bool graphs_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("FFB_GRAPHS");
    // the FFB_*_PROF probes synchronise inside the sequence: no capture then
    on = (e && atoi(e) == 0) || getenv("FFB_PIV_PROF") || getenv("FFB_PANEL_PROF") ||
                 getenv("FFB_JACOBI_PROF")
             ? 0
             : 1;
  }
  return on == 1;
}

template <typename T>
void key_put(std::string& k, const T& v) {
  k.append(reinterpret_cast<const char*>(&v), sizeof(v));
}

std::string graph_key(int mode, const double* A, int64_t lda, bool arow, int64_t m, int64_t n,
                      const Dims& D, const double* omega, const void* ws, size_t wsb,
                      const ffb_result* out) {
  std::string k;
  int dev = 0;
  cudaGetDevice(&dev);
  key_put(k, dev);
  key_put(k, mode);
  key_put(k, A);
  key_put(k, lda);
  key_put(k, arow);
  key_put(k, m);
  key_put(k, n);
  key_put(k, D.k);
  key_put(k, D.l);
  key_put(k, D.b);
  key_put(k, D.p);
  key_put(k, D.d);
  key_put(k, D.g);
  key_put(k, omega);
  key_put(k, ws);
  key_put(k, wsb);
  key_put(k, out->pivot_gap != nullptr);
  key_put(k, t_sm_budget);
  return k;
}

// Run `core` (a stream-ordered launch sequence with no host synchronisation) on
// `st`: replay its cached CUDA graph, or capture it on a private stream,
// instantiate, cache and launch it; anything not capturable runs eagerly.
template <class Eng_, class F>
void run_core(ffb_ctx* ctx, Eng_& e, cudaStream_t& st, const std::string& key, F&& core) {
  // graphs serve the one-problem-at-a-time path; batch worker threads (an SM
  // budget is set) launch eagerly: their launch latency is hidden by the other
  // problems in flight, and concurrent captures on many threads measured fragile
  if (!graphs_enabled() || t_sm_budget > 0) {
    core();
    return;
  }
  {
    std::lock_guard<std::mutex> g(ctx->gmu);
    auto it = ctx->graphs.find(key);
    if (it != ctx->graphs.end() && it->second.exec) {
      GraphEnt& ge = it->second;
      ge.stamp = ++ctx->gstamp;
      e.okm(cudaGraphLaunch(ge.exec, st));
      e.launches += ge.launches;
      e.gc.launches += ge.glaunches;
      e.gc.flops += ge.flops;
      return;
    }
    if (it == ctx->graphs.end()) {
      // first sighting: run eagerly (loads every kernel the sequence uses);
      // the second call with this key captures
      if (ctx->graphs.size() < kMaxGraphs) ctx->graphs.emplace(key, GraphEnt{});
      it = ctx->graphs.end();
      core();
      return;
    }
  }
  if (!begin_exclusive_capture()) {
    core();
    return;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  cudaStream_t& cap = t_host.capture[dev & 63];
  if (!cap && cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking) != cudaSuccess) {
    cap = nullptr;
    core();
    return;
  }
  const cudaStream_t user = st;
  const int64_t l0 = e.launches, gl0 = e.gc.launches, f0 = e.gc.flops;
  st = e.st = cap;
  cudaGraph_t graph = nullptr;
  struct EndCap {
    ~EndCap() { end_exclusive_capture(); }
  } end_cap;
  static const cudaStreamCaptureMode cmode = [] {
    const char* e = getenv("FFB_GRAPH_CAPTURE_MODE");   // 0 global, 1 thread-local, 2 relaxed
    const int v = e ? atoi(e) : 1;
    return v == 0 ? cudaStreamCaptureModeGlobal
                  : (v == 1 ? cudaStreamCaptureModeThreadLocal : cudaStreamCaptureModeRelaxed);
  }();
  bool ok = cudaStreamBeginCapture(cap, cmode) == cudaSuccess;
  if (ok) {
    core();
    const cudaError_t ce = cudaStreamEndCapture(cap, &graph);
    ok = ce == cudaSuccess && graph != nullptr && e.cerr == cudaSuccess;
  }
  st = e.st = user;
  cudaGraphExec_t exec = nullptr;
  if (ok) ok = cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess;
  if (graph) cudaGraphDestroy(graph);
  if (!ok) {   // not capturable here: run the sequence eagerly
    if (getenv("FFB_GRAPH_DEBUG"))
      fprintf(stderr, "[ffb graph] capture failed (%s), running eagerly\n",
              cudaGetErrorString(e.cerr != cudaSuccess ? e.cerr : cudaGetLastError()));
    (void)cudaGetLastError();
    e.cerr = cudaSuccess;
    e.launches = l0;
    e.gc.launches = gl0;
    e.gc.flops = f0;
    core();
    return;
  }
  GraphEnt ge;
  ge.exec = exec;
  ge.launches = e.launches - l0;
  ge.glaunches = e.gc.launches - gl0;
  ge.flops = e.gc.flops - f0;
  e.okm(cudaGraphLaunch(exec, st));
  std::lock_guard<std::mutex> g(ctx->gmu);
  auto found = ctx->graphs.find(key);
  if (found != ctx->graphs.end() && found->second.exec) {   // captured meanwhile elsewhere
    ctx->retired.push_back(exec);
    return;
  }
  if (found == ctx->graphs.end() && ctx->graphs.size() >= kMaxGraphs) {
    auto old = ctx->graphs.begin();
    for (auto it = ctx->graphs.begin(); it != ctx->graphs.end(); ++it)
      if (it->second.stamp < old->second.stamp) old = it;
    if (old->second.exec) {
      cudaDeviceSynchronize();   // the evicted graph may still run on another stream
      cudaGraphExecDestroy(old->second.exec);
    }
    ctx->graphs.erase(old);
  }
  ge.stamp = ++ctx->gstamp;
  ctx->graphs[key] = ge;
}

bool validate(const Dims& D) {
  if (D.m < 1 || D.n < 1) return false;
  if (!(1 <= D.k && D.k <= D.l && D.l <= std::min(D.m, D.n))) return false;
  if (D.b < 1 || D.p < 0 || D.s > D.m) return false;
  if (D.d < 1 || D.d > D.l) return false;
  if (D.mode != FFB_MODE_TRQRCP && D.l + 1 > std::min(D.m, D.n)) return false;
  if (D.s > 512) return false;  // pivot kernel: winner column <= 16 rows per lane of one warp
  if (D.n >= 2147483647LL) return false;  // pivot exchange carries 32-bit positions
  return true;
}

}  // namespace

extern "C" {

const char* ffb_version(void) { return "ffb200 0.1.0 (sm_100a, FP64 DMMA)"; }

int ffb_ctx_create(int device, ffb_ctx** out) {
  if (!out) return FFB_ERR_ARGUMENT;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) return FFB_ERR_CUDA;
  DeviceGuard dg(device);
  ffb_ctx* c = new ffb_ctx();
  c->device = device;
  cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device);
  cudaMallocHost(&c->sc_host, sizeof(SrqrScalars));
  *out = c;
  return FFB_OK;
}

int ffb_ctx_destroy(ffb_ctx* c) {
  if (!c) return FFB_OK;
  {
    DeviceGuard dg(c->device);
    cudaDeviceSynchronize();
    for (auto& kv : c->graphs)
      if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    for (auto ex : c->retired) cudaGraphExecDestroy(ex);
  }
  if (c->pinned) cudaFreeHost(c->pinned);
  if (c->sc_host) cudaFreeHost(c->sc_host);
  delete c;
  return FFB_OK;
}

const char* ffb_last_error(const ffb_ctx* c) {
  (void)c;
  return t_err.c_str();
}

int ffb_workspace_query(int64_t m, int64_t n, const ffb_params* prm, int mode, size_t* bytes) {
  if (!prm || !bytes) return FFB_ERR_ARGUMENT;
  Dims D{m, n, prm->k, prm->l, prm->b, prm->p, prm->b + prm->p, prm->d, prm->g, prm->seed, mode};
  if (!validate(D)) return FFB_ERR_DIMENSION;
  Work w;
  *bytes = carve(nullptr, D, nullptr, (size_t)-1, w) + (8u << 20);
  return FFB_OK;
}

int ffb_gemm(ffb_ctx* ctx, void* stream, int64_t M, int64_t N, int64_t K, double alpha,
             const double* A, int64_t lda, int a_kc, const double* B, int64_t ldb, int b_kc,
             double beta, double* C, int64_t ldc, void* workspace, size_t workspace_bytes) {
  if (!ctx) return FFB_ERR_ARGUMENT;
  DeviceGuard dg(ctx->device);
  GemmCtx gc;
  CallGuard call_guard;
  gc.sms = ctx->sms;
  // workspace: [stream-K counters (64Ki u32, zeroed here) | split-K / stream-K partials]
  const size_t cnt_bytes = 65536 * sizeof(unsigned);
  if (workspace && workspace_bytes > cnt_bytes + 4096) {
    gc.counters = static_cast<unsigned*>(workspace);
    gc.counter_cap = 65536;
    cudaMemsetAsync(workspace, 0, cnt_bytes, (cudaStream_t)stream);
    gc.partial = reinterpret_cast<double*>(static_cast<char*>(workspace) + cnt_bytes);
    gc.partial_cap = (workspace_bytes - cnt_bytes) / sizeof(double);
  }
  cudaError_t e = gemm_f64(gc, (cudaStream_t)stream, M, N, K, alpha, A, lda, a_kc != 0, B, ldb,
                           b_kc != 0, beta, C, ldc);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "ffb_gemm");
  return FFB_OK;
}

int ffb_block_pivots(ffb_ctx* ctx, void* stream, const double* B, int64_t s, int64_t n,
                     int64_t ldb, int64_t j0, int64_t bb, int64_t* arr, int64_t* pos, double* gap,
                     void* workspace, size_t workspace_bytes) {
  if (!ctx) return FFB_ERR_ARGUMENT;
  DeviceGuard dg(ctx->device);
  CallGuard call_guard;
  if (bb < 1 || j0 < 0 || j0 + bb > n || n >= 2147483647LL || s < 1 || s > 512)
    return fail(ctx, FFB_ERR_DIMENSION, "bad pivot block");
  Work w;
  pivot_geometry(ctx, n, s, w);
  Bump b{static_cast<char*>(workspace), 0, workspace_bytes};
  w.prec = b.take<unsigned long long>(2 * (size_t)w.G * pivots_recw((int)s));
  w.hist = b.take<int64_t>(bb);
  w.pwork = w.piv_smem ? nullptr : b.take<double>((size_t)w.G * pivots_stride((int)s) * w.cpc);
  if (!b.ok) return fail(ctx, FFB_ERR_ARGUMENT, "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(w.prec, 0, 16 * (size_t)w.G * pivots_recw((int)s), st);
  PivotArgs a{B, ldb, (int)s, n, j0, (int)bb, arr, pos, w.G, w.cpc, 0, w.pwork, w.prec,
              pivots_recw((int)s), w.hist, gap};
  if (e == cudaSuccess) {
    e = launch_pivots(st, a, w.piv_smem, w.piv_smem_bytes);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "ffb_block_pivots");
  return FFB_OK;
}

int ffb_run(ffb_ctx* ctx, void* stream, int mode, const double* A, int64_t m, int64_t n,
            int64_t lda, int a_layout, const ffb_params* prm, const double* omega,
            ffb_gauss_cb gauss, void* gauss_user, void* workspace, size_t workspace_bytes,
            ffb_result* out) {
  if (!ctx || !prm || !out || !A || !omega || !workspace) return FFB_ERR_ARGUMENT;
  CallGuard call_guard;
  if (a_layout != FFB_LAYOUT_COL && a_layout != FFB_LAYOUT_ROW) return FFB_ERR_ARGUMENT;
  const AView av{A, lda, a_layout == FFB_LAYOUT_ROW};
  DeviceGuard dg(ctx->device);
  Eng e;
  e.ctx = ctx;
  e.st = (cudaStream_t)stream;
  Dims& D = e.D;
  D = Dims{m, n, prm->k, prm->l, prm->b, prm->p, prm->b + prm->p, prm->d, prm->g, prm->seed, mode};
  if (!validate(D) || lda < (av.row ? n : m))
    return fail(ctx, FFB_ERR_DIMENSION, "invalid dimensions/parameters");
  if (mode == FFB_MODE_FLIPFLOP && (!out->u || !out->s || !out->v))
    return fail(ctx, FFB_ERR_ARGUMENT, "u, s, v outputs are required");
  Work& w = e.w;
  const size_t need = carve(ctx, D, workspace, workspace_bytes, w);
  if (need > workspace_bytes) return fail(ctx, FFB_ERR_ARGUMENT, "workspace too small");
  e.sms = effective_sms(ctx);
  // GEMMs are not grid-synchronised: their split / stream-K choices stay those of
  // the whole device, so results do not depend on the caller's SM budget
  e.gc.sms = ctx->sms;
  e.gc.partial = w.gpart;
  e.gc.partial_cap = w.gpart_cap;
  e.gc.counters = w.skcnt;
  e.gc.counter_cap = 65536;
  cudaStream_t st = e.st;
  const int64_t l = D.l, s = D.s, L1 = l + 1;

  // g2 test matrix for swaps == 0 (stream 1000), generated on the host by the
  // reference's RNG and staged now so the pipeline never waits for the host.
  auto stage_gauss = [&](int64_t swaps) -> int {
    const size_t cnt = (size_t)D.d * L1;
    if (t_host.cap < cnt) {
      if (t_host.pinned) cudaFreeHost(t_host.pinned);
      cudaMallocHost(&t_host.pinned, cnt * sizeof(double));
      t_host.cap = cnt;
    }
    cudaStreamSynchronize(st);  // previous staging copy may still read the buffer
    if (!gauss || gauss(gauss_user, D.seed, 1000 + (uint64_t)swaps, D.d, L1, t_host.pinned) != 0)
      return fail(ctx, FFB_ERR_ARGUMENT, "gauss callback failed");
    e.ok(launch_copy_bytes(st, t_host.pinned, w.g2om, cnt * sizeof(double)));   // reads pinned host memory (UVA)
    return FFB_OK;
  };
  if (mode != FFB_MODE_TRQRCP) {
    int rc = stage_gauss(0);
    if (rc) return rc;
  }

  // ---------------------------------------------------------------- TRQRCP
  auto trqrcp_body = [&]() {
    e.okm(cudaMemsetAsync(w.status, 0, sizeof(uint32_t), st));
    e.okm(cudaMemsetAsync(w.skcnt, 0, sizeof(unsigned) * 65536, st));
    // B = Omega * A (Omega row-major s x m: A-operand with contiguous k)
    e.gemm(s, n, m, 1.0, omega, m, true, A, lda, av.kc_as_b(), 0.0, w.B, s);
    if (av.row) e.ok(launch_colsq_rm(st, A, lda, m, n, w.cpart, w.colsq));
    else e.ok(launch_colsq(st, A, lda, m, n, w.colsq));
    e.ok(launch_finite_check(st, w.colsq, (size_t)n, w.status));   // NaN / Inf anywhere in A
    e.ok(launch_iota2(st, w.arr, w.pos, n));
    e.memset2d(w.Y, m, m, l);
    e.memset2d(w.T, l, l, l);
    e.memset2d(w.WT, l, l, n);
    e.memset2d(w.R, L1, L1, n);
    {
    }
    for (int64_t j0 = 0; j0 < l && e.cerr == cudaSuccess; j0 += D.b) {
      const int64_t bb = std::min<int64_t>(D.b, l - j0), e1 = j0 + bb;
      // (K2) pivots on the sketch
      e.okm(cudaMemsetAsync(w.prec, 0, 16 * (size_t)w.G * pivots_recw((int)s), st));
      PivotArgs pa{w.B, s, (int)s, n, j0, (int)bb, w.arr, w.pos, w.G, w.cpc, 0, w.pwork, w.prec,
                   pivots_recw((int)s), w.hist, out->pivot_gap ? w.gap + j0 : nullptr};
      e.ok(launch_pivots(st, pa, w.piv_smem, w.piv_smem_bytes));
      // (K4) panel P = A[:, piv] - Y[:, :j0] WT[:j0, piv]
      e.ok(launch_gather_cols_strided(st, A, av.rs(), av.cs(), m, w.arr + j0, bb, w.P, m));
      if (j0 > 0) {
        e.ok(launch_gather_cols(st, w.WT, l, j0, w.arr + j0, bb, w.WTg, j0));
        e.gemm(m, bb, j0, -1.0, w.Y, m, false, w.WTg, j0, true, 1.0, w.P, m);
      }
      // Householder QR of P[j0:, :] -> Y block, T block, Rb
      e.hh_qr(w.P + j0, m - j0, bb, m, w.Y + j0 + j0 * m, m, w.T + j0 + j0 * l, l, w.Rb, bb, true);
      // T12 = -T11 (Y1^T Y2) T22
      if (j0 > 0) {
        e.gemm(j0, bb, m - j0, 1.0, w.Y + j0, m, true, w.Y + j0 + j0 * m, m, true, 0.0, w.S1, j0);
        e.gemm(j0, bb, bb, 1.0, w.S1, j0, false, w.T + j0 + j0 * l, l, true, 0.0, w.S2, j0);
        e.gemm(j0, bb, j0, -1.0, w.T, l, false, w.S2, j0, true, 0.0, w.T + j0 * l, l);
      }
      // (K5) WT[j0:e, :] = T22^T (Y2^T A - (Y2^T Y1) WT[:j0, :])
      e.gemm(bb, n, m - j0, 1.0, w.Y + j0 + j0 * m, m, true, av.rows_from(j0), lda, av.kc_as_b(), 0.0,
             w.G1, bb);
      if (j0 > 0) e.gemm(bb, n, j0, -1.0, w.S1, j0, true, w.WT, l, true, 1.0, w.G1, bb);
      e.gemm(bb, n, bb, 1.0, w.T + j0 + j0 * l, l, true, w.G1, bb, true, 0.0, w.WT + j0, l);
      // (K6) R[j0:e, :] = A[j0:e, :] - Y[j0:e, :e] WT[:e, :]
      if (av.row) e.ok(launch_copy_rows_rm(st, av.rows_from(j0), lda, bb, n, w.R + j0, L1));
      else e.ok(launch_copy_rows(st, A + j0, lda, bb, n, w.R + j0, L1));
      e.gemm(bb, n, e1, -1.0, w.Y + j0, m, false, w.WT, l, true, 1.0, w.R + j0, L1);
      e.ok(launch_fix_rrows(st, w.R, L1, j0, (int)bb, w.arr, w.Rb, bb));
      // sketch update B[:, trailing] -= (B_piv R11^{-1}) R12
      if (e1 < n) {
        e.ok(launch_gather_cols(st, w.B, s, s, w.arr + j0, bb, w.Bp, s));
        e.tri_inverse(w.Rb, bb, bb, w.Rinv, bb);
        e.gemm(s, bb, bb, 1.0, w.Bp, s, false, w.Rinv, bb, true, 0.0, w.Z, s);
        e.gemm(s, n, bb, -1.0, w.Z, s, false, w.R + j0, L1, true, 1.0, w.B, s);
      }
    }
  };

  auto outputs_common = [&]() {
    if (out->perm)
      e.ok(d2d(out->perm, w.arr, sizeof(int64_t) * n, st));
    if (out->R) e.ok(launch_r_arranged(st, w.R, L1, w.arr, l, n, out->R, out->ldr, l));
    if (out->B) e.ok(launch_gather_cols(st, w.B, s, s, w.arr, n, out->B, out->ldb));
    if (out->pivot_gap)
      e.ok(d2d(out->pivot_gap, w.gap, sizeof(double) * l, st));
  };

  // ------------------------------------------------------------------ SRQR
  auto srqr_init = [&]() {
    // dense Q[:, :l] = E - Y (T Y[:l, :]^T)   (srqr.py:91-93)
    e.gemm(l, l, l, 1.0, w.T, l, false, w.Y, m, false, 0.0, w.TYt, l);
    e.gemm(m, l, l, -1.0, w.Y, m, false, w.TYt, l, true, 0.0, w.Q, m);
    e.ok(launch_add_identity(st, w.Q, m, m, l, 1.0));
    e.okm(cudaMemsetAsync(w.Q + m * l, 0, sizeof(double) * m, st));
    e.ok(launch_rinit(st, w.B, s, (int)s, w.arr, n, l, w.r, w.rinit));
    e.ok(launch_anorm(st, w.colsq, n, w.sc));
  };
  auto extend = [&]() {
    e.ok(launch_ext_pick(st, l, n, w.arr, w.pos, w.r, w.rinit, w.sc));
    e.ok(launch_ext_project(st, A, av.rs(), av.cs(), m, l, w.Q, m, w.R, L1, w.arr, w.u, w.ct, w.part,
                            w.sc, w.r, w.R));
    const int nparts = (int)((m + 255) / 256);
    e.ok(launch_ext_finish(st, w.part, nparts, l, n, w.arr, w.R, L1, w.r, w.sc, w.u, m, w.Q + m * l));
  };

  auto pack = [&]() { e.ok(launch_pack(st, w.R, L1, w.arr, w.colsq, l, n, w.part, 0, w.sc)); };
  auto pack_outputs = [&]() {
    outputs_common();
    if (out->Q) e.ok(launch_copy_rows(st, w.Q, m, m, L1, out->Q, out->ldq));
    if (out->rtilde) e.ok(launch_r_arranged(st, w.R, L1, w.arr, L1, L1, out->rtilde, L1, L1));
  };

  // ------------------------------------------------------------ flip-flop
  auto flipflop_core = [&]() {
    e.ok(launch_build_rt(st, w.R, L1, w.arr, l, n, w.X, n));
    e.hh_qr(w.X, n, l, n, w.Yl, n, w.Tl, l, w.Rl, l, false);
    // Qhat1 = E - Yl (Tl Yl[:l,:]^T) ; Yh = Pi Qhat1 (rows scattered to original order)
    e.gemm(l, l, l, 1.0, w.Tl, l, false, w.Yl, n, false, 0.0, w.TYt, l);
    e.gemm(n, l, l, -1.0, w.Yl, n, false, w.TYt, l, true, 0.0, w.Qh, n);
    e.ok(launch_add_identity(st, w.Qh, n, n, l, 1.0));
    e.ok(launch_scatter_rows(st, w.Qh, n, n, l, w.arr, w.Yh, n));
    // (K13) tmp = A * Yh
    e.gemm(m, l, n, 1.0, A, lda, av.kc_as_a(), w.Yh, n, true, 0.0, w.tmp, m);
    // (K14) tmp = Qt Rt, SVD(Rt)
    e.hh_qr(w.tmp, m, l, m, w.Yt, m, w.Tt, l, w.Rt, l, true);
    // one-sided block Jacobi SVD of Rt (ffb_jacobi.cu): Rt = Us diag(sig) Vo^T
    e.ok(launch_jacobi_svd(st, e.sms, w.Rt, l, (int)l, w.sig, w.Us, l, w.Vo, l, w.jwork, w.jbar,
                           w.joff, w.jsweeps, w.jorder, kMaxSweeps));
    e.launches += 5;   // scale, layout, Jacobi, V replay, norms, out kernels
    // (K15, left half) W2 = Tt (Yt[:l]^T Us[:, :k])
    e.gemm(l, D.k, l, 1.0, w.Yt, m, true, w.Us, l, true, 0.0, w.W1, l);
    e.gemm(l, D.k, l, 1.0, w.Tt, l, false, w.W1, l, true, 0.0, w.W2, l);
  };
  // the caller's outputs of the flip-flop tail (kept out of the cached graph so
  // its key does not depend on where the caller's output buffers live)
  auto flipflop_out = [&]() {
    const int64_t k = D.k;
    if (out->diag_L) e.ok(launch_diag(st, w.Rl, l, l, out->diag_L));
    // (K15) u = Qt[:, :l] Us[:, :k] ; v = Yh Vs[:, :k]
    e.gemm(m, k, l, -1.0, w.Yt, m, false, w.W2, l, true, 0.0, out->u, out->ldu);
    e.ok(launch_add_top(st, out->u, out->ldu, w.Us, l, l, k));
    e.gemm(n, k, l, 1.0, w.Yh, n, false, w.Vo, l, true, 0.0, out->v, out->ldv);
    e.ok(d2d(out->s, w.sig, sizeof(double) * k, st));
    if (out->sv_all) e.ok(d2d(out->sv_all, w.sig, sizeof(double) * l, st));
  };

  // The launch sequence up to the certificate depends only on the shapes, the
  // parameters and the device buffers (A, Omega, workspace): it is captured once
  // into a CUDA graph and replayed by later calls with the same key.
  auto core = [&]() {
    trqrcp_body();
    if (mode == FFB_MODE_TRQRCP) return;
    srqr_init();
    extend();
    e.g2();
    pack();
    if (mode == FFB_MODE_FLIPFLOP) flipflop_core();
  };
  run_core(ctx, e, st, graph_key(mode, A, lda, av.row, m, n, D, omega, workspace, workspace_bytes, out),
           core);

  if (mode == FFB_MODE_TRQRCP) {
    outputs_common();
    if (out->Y) e.ok(launch_copy_rows(st, w.Y, m, m, l, out->Y, out->ldy));
    if (out->T) e.ok(launch_copy_rows(st, w.T, l, l, l, out->T, out->ldt));
    cudaError_t se = cudaStreamSynchronize(st);
    if (e.cerr != cudaSuccess) return cuda_fail(ctx, e.cerr, "trqrcp launch");
    if (se != cudaSuccess) return cuda_fail(ctx, se, "trqrcp");
    uint32_t stw = 0;
    d2h(&stw, w.status, sizeof(stw), st);
    ++e.launches;   // d2h's copy kernel
    out->status_bits = stw;
    out->flops = e.gc.flops;
    out->kernels = e.gc.launches + e.launches;
    if (stw & (kStNonFinite | kStCholFail)) return fail(ctx, FFB_ERR_NUMERICAL, "numerical failure in TRQRCP");
    return FFB_OK;
  }

  pack_outputs();
  if (mode == FFB_MODE_FLIPFLOP) flipflop_out();

  auto read_sc = [&]() -> cudaError_t {
    if (!t_host.sc) cudaMallocHost(&t_host.sc, sizeof(SrqrScalars));
    e.ok(launch_copy_bytes(st, w.sc, t_host.sc, sizeof(SrqrScalars)));   // writes pinned host memory (UVA)
    return cudaStreamSynchronize(st);
  };
  cudaError_t se = read_sc();
  if (e.cerr != cudaSuccess) return cuda_fail(ctx, e.cerr, "launch");
  if (se != cudaSuccess) return cuda_fail(ctx, se, "srqr");
  SrqrScalars sc = *t_host.sc;
  uint32_t stw = 0;
  d2h(&stw, w.status, sizeof(stw), st);
  ++e.launches;
  stw |= sc.status;
  out->status_bits = stw;
  if (stw & kStNonFinite) return fail(ctx, FFB_ERR_NUMERICAL, "non-finite values in input or factors");
  if (stw & kStCholFail) return fail(ctx, FFB_ERR_NUMERICAL, "panel CholeskyQR breakdown (rank-deficient panel)");
  if (stw & kStSingular) return fail(ctx, FFB_ERR_SINGULAR_TRAILING, "zero diagonal in leading triangular block");

  int64_t swaps = 0;
  if (sc.need_swap) {
    // ---- the reference's swap loop (srqr.py:192-206), host-driven
    while (true) {
      if (swaps >= 50 * l) {
        pack();
        pack_outputs();
        se = read_sc();
        sc = *t_host.sc;
        out->alpha = sc.alpha; out->g1 = sc.g1; out->g2 = sc.g2; out->r22 = sc.r22;
        out->tau_bound = sc.tau; out->tau_hat_bound = sc.tau_hat; out->swaps = swaps;
        return fail(ctx, FFB_ERR_CERTIFICATION, "swap cap reached");
      }
      e.ok(launch_ext_row(st, A, av.rs(), av.cs(), m, n, l, w.Q, m, w.R, L1, w.arr, w.colsq, w.r,
                          w.rinit, w.sc));
      if (swaps < 64) out->i_off_trace[swaps] = sc.i_off;
      ++swaps;
      e.ok(launch_rotate_out(st, w.R, L1, w.Q, m, m, n, l, w.arr, w.pos, w.r, w.rinit, w.sc, w.rot));
      e.ok(launch_revert(st, w.R, L1, w.arr, l, n, w.r));
      extend();
      se = read_sc();
      if (e.cerr != cudaSuccess || se != cudaSuccess) return cuda_fail(ctx, e.cerr ? e.cerr : se, "swap");
      sc = *t_host.sc;
      if (!(sc.alpha > 0.0)) break;
      int rc = stage_gauss(swaps);
      if (rc) return rc;
      e.g2();
      se = read_sc();
      if (e.cerr != cudaSuccess || se != cudaSuccess) return cuda_fail(ctx, e.cerr ? e.cerr : se, "swap g2");
      sc = *t_host.sc;
      if (sc.status & kStSingular) return fail(ctx, FFB_ERR_SINGULAR_TRAILING, "zero diagonal in leading triangular block");
      if (!sc.need_swap) break;
    }
    pack();
    pack_outputs();
    if (mode == FFB_MODE_FLIPFLOP) {
      flipflop_core();
      flipflop_out();
    }
    se = read_sc();
    if (e.cerr != cudaSuccess) return cuda_fail(ctx, e.cerr, "launch");
    if (se != cudaSuccess) return cuda_fail(ctx, se, "flipflop");
    sc = *t_host.sc;
  }
  if (mode == FFB_MODE_FLIPFLOP) {
    int sweeps = 0;
    d2h(&sweeps, w.jsweeps, sizeof(int), st);
    ++e.launches;
    out->svd_sweeps = sweeps;
    if (sweeps >= kMaxSweeps) return fail(ctx, FFB_ERR_NUMERICAL, "small SVD did not converge");
  }
  out->alpha = sc.alpha;
  out->g1 = sc.g1;
  out->g2 = sc.alpha > 0.0 ? sc.g2 : 0.0;
  out->r22 = sc.r22;
  out->tau_bound = sc.tau;
  out->tau_hat_bound = sc.tau_hat;
  out->swaps = swaps;
  out->flops = e.gc.flops;
  out->kernels = e.gc.launches + e.launches;
  return FFB_OK;
}

int ffb_flipflop(ffb_ctx* ctx, void* stream, const double* A, int64_t m, int64_t n, int64_t lda,
                 int a_layout, const ffb_params* prm, const double* omega, ffb_gauss_cb gauss,
                 void* gauss_user, void* workspace, size_t workspace_bytes, ffb_result* out) {
  return ffb_run(ctx, stream, FFB_MODE_FLIPFLOP, A, m, n, lda, a_layout, prm, omega, gauss,
                 gauss_user, workspace, workspace_bytes, out);
}

}  // extern "C"

extern "C" int ffb_set_thread_sm_budget(int sms) {
  t_sm_budget = sms > 0 ? sms : 0;
  return FFB_OK;
}

extern "C" int ffb_run_batched(ffb_ctx* ctx, ffb_batch_item* items, int64_t count, int max_threads,
                               ffb_gauss_cb gauss, void* gauss_user) {
  if (!ctx || (count > 0 && !items)) return FFB_ERR_ARGUMENT;
  if (count <= 0) return FFB_OK;
  int nt = max_threads < 1 ? 1 : max_threads;
  if (nt > count) nt = (int)count;
  std::atomic<int64_t> next{0};
  std::vector<std::string> msgs((size_t)count);
  const int budget = nt > 1 ? std::max(8, ctx->sms / nt) : 0;
  auto worker = [&]() {
    const int saved = t_sm_budget;
    if (budget) t_sm_budget = budget;
    for (int64_t i = next++; i < count; i = next++) {
      ffb_batch_item& it = items[i];
      it.status = ffb_run(ctx, it.stream, it.mode, it.A, it.m, it.n, it.lda, it.a_layout, &it.prm,
                          it.omega, gauss, gauss_user, it.workspace, it.workspace_bytes, it.out);
      if (it.status != FFB_OK) msgs[(size_t)i] = t_err;
    }
    t_sm_budget = saved;
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < nt; ++t) pool.emplace_back(worker);
  worker();
  for (auto& t : pool) t.join();
  for (int64_t i = 0; i < count; ++i)
    if (items[i].status != FFB_OK) {
      t_err = "problem " + std::to_string(i) + ": " + msgs[(size_t)i];
      return items[i].status;
    }
  return FFB_OK;
}

// --------------------------------------------------------------------------
// Randomized subspace-iteration SVD (the paper's RSISVD baseline,
// ffsrqr/svd.py:101-133): Y = A Omega; Q = qr(Y); q times { Q = qr(A^T Q);
// Q = qr(A Q) }; B = Q^T A; SVD(B) through B^T = Q_b R_b and the one-sided
// Jacobi SVD of R_b (R_b = U_r S V_r^T => B = V_r S (Q_b U_r)^T).  All QRs are
// the Householder panels of the flip-flop path (LAPACK dgeqrf/dorgqr convention,
// so Q equals numpy.linalg.qr's up to rounding); u, v match LAPACK dgesdd's up
// to column signs.
extern "C" int ffb_rsisvd_workspace_query(int64_t m, int64_t n, int64_t k, int64_t r,
                                          size_t* bytes) {
  if (!bytes) return FFB_ERR_ARGUMENT;
  if (m < 1 || n < 1 || k < 1 || k > r || r > std::min(m, n)) return FFB_ERR_DIMENSION;
  Work w;
  *bytes = carve_rsisvd(nullptr, m, n, k, r, nullptr, (size_t)-1, w) + (8u << 20);
  return FFB_OK;
}

extern "C" int ffb_rsisvd(ffb_ctx* ctx, void* stream, const double* A, int64_t m, int64_t n,
                          int64_t lda, int a_layout, int64_t k, int64_t r, int64_t q, const double* omega,
                          void* workspace, size_t workspace_bytes, double* u, int64_t ldu,
                          double* s, double* v, int64_t ldv, int64_t* flops, int32_t* sweeps_out) {
  if (!ctx || !A || !omega || !workspace || !u || !s || !v) return FFB_ERR_ARGUMENT;
  CallGuard call_guard;
  DeviceGuard dg(ctx->device);
  if (a_layout != FFB_LAYOUT_COL && a_layout != FFB_LAYOUT_ROW) return FFB_ERR_ARGUMENT;
  const bool arow = a_layout == FFB_LAYOUT_ROW;
  if (m < 1 || n < 1 || k < 1 || k > r || r > std::min(m, n) || q < 0 || lda < (arow ? n : m) ||
      ldu < m || ldv < n)
    return fail(ctx, FFB_ERR_DIMENSION, "rsisvd needs 1 <= k <= r <= min(m, n), q >= 0");
  Eng e;
  e.ctx = ctx;
  e.st = (cudaStream_t)stream;
  Work& w = e.w;
  const size_t need = carve_rsisvd(ctx, m, n, k, r, workspace, workspace_bytes, w);
  if (need > workspace_bytes) return fail(ctx, FFB_ERR_ARGUMENT, "workspace too small");
  e.sms = effective_sms(ctx);
  // GEMMs are not grid-synchronised: their split / stream-K choices stay those of
  // the whole device, so results do not depend on the caller's SM budget
  e.gc.sms = ctx->sms;
  e.gc.partial = w.gpart;
  e.gc.partial_cap = w.gpart_cap;
  e.gc.counters = w.skcnt;
  e.gc.counter_cap = 65536;
  cudaStream_t st = e.st;
  e.okm(cudaMemsetAsync(w.status, 0, sizeof(uint32_t), st));
  e.okm(cudaMemsetAsync(w.skcnt, 0, sizeof(unsigned) * 65536, st));
  // Y = A Omega (Omega n x r, row-major = numpy C order)
  e.gemm(m, r, n, 1.0, A, lda, arow, omega, r, false, 0.0, w.tmp, m);
  e.hh_qr(w.tmp, m, r, m, w.Yt, m, w.Tt, r, w.Rt, r, false);
  explicit_q(e, w.Yt, m, w.Tt, r, m, r, w.Q, m);
  for (int64_t it = 0; it < q; ++it) {
    e.gemm(n, r, m, 1.0, A, lda, !arow, w.Q, m, true, 0.0, w.X, n);         // Z = A^T Q
    e.hh_qr(w.X, n, r, n, w.Yl, n, w.Tl, r, w.Rl, r, false);
    explicit_q(e, w.Yl, n, w.Tl, r, n, r, w.Qh, n);
    e.gemm(m, r, n, 1.0, A, lda, arow, w.Qh, n, true, 0.0, w.tmp, m);       // Y = A Q_z
    e.hh_qr(w.tmp, m, r, m, w.Yt, m, w.Tt, r, w.Rt, r, false);
    explicit_q(e, w.Yt, m, w.Tt, r, m, r, w.Q, m);
  }
  // B^T = A^T Q = Q_b R_b
  e.gemm(n, r, m, 1.0, A, lda, !arow, w.Q, m, true, 0.0, w.X, n);
  e.hh_qr(w.X, n, r, n, w.Yl, n, w.Tl, r, w.Rl, r, true);
  e.ok(launch_jacobi_svd(st, e.sms, w.Rl, r, (int)r, w.sig, w.Us, r, w.Vo, r, w.jwork, w.jbar,
                         w.joff, w.jsweeps, w.jorder, kMaxSweeps));
  e.launches += 5;
  // u = Q V_r[:, :k] ; v = Q_b [U_r[:, :k]; 0] ; s = sigma[:k]
  e.gemm(m, k, r, 1.0, w.Q, m, false, w.Vo, r, true, 0.0, u, ldu);
  e.gemm(r, k, r, 1.0, w.Yl, n, true, w.Us, r, true, 0.0, w.W1, r);
  e.gemm(r, k, r, 1.0, w.Tl, r, false, w.W1, r, true, 0.0, w.W2, r);
  e.gemm(n, k, r, -1.0, w.Yl, n, false, w.W2, r, true, 0.0, v, ldv);
  e.ok(launch_add_top(st, v, ldv, w.Us, r, r, k));
  e.ok(d2d(s, w.sig, sizeof(double) * k, st));
  int sw = 0;
  uint32_t stw = 0;
  cudaError_t se = cudaSuccess;
  if (e.cerr == cudaSuccess) se = d2h(&sw, w.jsweeps, sizeof(int), st);
  if (e.cerr == cudaSuccess && se == cudaSuccess) se = d2h(&stw, w.status, sizeof(stw), st);
  e.launches += 2;   // the two d2h copy kernels
  if (e.cerr != cudaSuccess) return cuda_fail(ctx, e.cerr, "rsisvd launch");
  if (se != cudaSuccess) return cuda_fail(ctx, se, "rsisvd");
  if (flops) *flops = e.gc.flops;
  if (sweeps_out) *sweeps_out = sw;
  if (stw & 1u) return fail(ctx, FFB_ERR_NUMERICAL, "non-finite values in rsisvd");
  if (sw >= kMaxSweeps) return fail(ctx, FFB_ERR_NUMERICAL, "small SVD did not converge");
  return FFB_OK;
}

// --------------------------------------------------------------------------
// Standalone small SVD (the dgesdd of svd.py:79): the flip-flop's Jacobi.
namespace {
size_t carve_small_svd(int64_t l, void* base, size_t cap, Work& w) {
  Bump b{static_cast<char*>(base), 0, cap};
  w.jwork = b.take<double>(jacobi_work_doubles((int)l, kMaxSweeps));
  w.joff = b.take<double>(kMaxSweeps);
  w.jbar = b.take<uint32_t>(4);
  w.jsweeps = b.take<int>(4);
  w.jorder = b.take<int>(l);
  return b.off + kAlign;
}
}  // namespace

extern "C" int ffb_small_svd_workspace_query(int64_t l, size_t* bytes) {
  if (!bytes) return FFB_ERR_ARGUMENT;
  if (l < 1 || l > (1 << 20)) return FFB_ERR_DIMENSION;
  Work w;
  *bytes = carve_small_svd(l, nullptr, (size_t)-1, w);
  return FFB_OK;
}

extern "C" int ffb_small_svd(ffb_ctx* ctx, void* stream, const double* M, int64_t l, int64_t ldm,
                             double* sig, double* U, int64_t ldu, double* V, int64_t ldv,
                             void* workspace, size_t workspace_bytes, int32_t* sweeps) {
  if (!ctx || !M || !sig || !U || !V || !workspace) return FFB_ERR_ARGUMENT;
  CallGuard call_guard;
  DeviceGuard dg(ctx->device);
  if (l < 1 || ldm < l || ldu < l || ldv < l) return fail(ctx, FFB_ERR_DIMENSION, "small svd needs l >= 1, ld >= l");
  Work w;
  if (carve_small_svd(l, workspace, workspace_bytes, w) > workspace_bytes)
    return fail(ctx, FFB_ERR_ARGUMENT, "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = launch_jacobi_svd(st, effective_sms(ctx), M, ldm, (int)l, sig, U, ldu, V, ldv, w.jwork, w.jbar,
                                    w.joff, w.jsweeps, w.jorder, kMaxSweeps);
  int sw = 0;
  if (e == cudaSuccess) e = d2h(&sw, w.jsweeps, sizeof(int), st);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "ffb_small_svd");
  if (sweeps) *sweeps = sw;
  if (sw >= kMaxSweeps) return fail(ctx, FFB_ERR_NUMERICAL, "small SVD did not converge");
  return FFB_OK;
}
