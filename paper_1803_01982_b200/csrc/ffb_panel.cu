// Fused Householder panel factorization (K4 / K12 building block), one
// cooperative launch per panel of width w <= 64:
//
//   shifted CholeskyQR3 of X (Mp x w)   [Fukaya et al. 2020]
//     pass p: local Gram of each CTA's rows (smem-staged, FP64)  -> partials
//             grid barrier -> distributed fixed-order reduction -> grid barrier
//             every CTA: Cholesky + triangular inverse of the Gram (redundant,
//             so no broadcast step), rows <- rows * R^-1
//   Householder reconstruction [Ballard et al.]: LU of Q_top*D - I with the sign
//   D_c that makes every pivot <= -1 (the reference's alpha = -sign(x0)||x||,
//   ffsrqr/qr.py:21-43), Y = [L; Q_bottom * D U^-1], T = -U L^-T, R = D * Racc.
//
// Results are deterministic (fixed reduction order).  Replaces 11-14 launches of
// GEMM + single-CTA kernels per panel.
#include <math.h>

#include "ffb_common.cuh"
#include "ffb_panel.cuh"

namespace ffb {

namespace {

constexpr int kW = 64;
constexpr int kL = kW + 1;   // padded leading dimension in shared memory
constexpr int kCH = 64;      // rows per staged chunk

FFB_DEV uint32_t ld_acq32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
FFB_DEV void st_rel32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

FFB_DEV void grid_sync(uint32_t* bar, uint32_t nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t gen = ld_acq32(bar + 1);
    __threadfence();
    const uint32_t arrived = atomicAdd(bar, 1u) + 1u;
    if (arrived == nblocks) {
      atomicExch(bar, 0u);
      __threadfence();
      st_rel32(bar + 1, gen + 1u);
    } else {
      while (ld_acq32(bar + 1) == gen) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

// Cholesky (upper, R^T R = G) of the w x w Gram in Gs (destroyed), R into Rs,
// X = R^-1 into Xs.  256 threads.  Returns false on breakdown.
FFB_DEV bool chol_inv(double* Gs, double* Rs, double* Xs, int w, double shift_coef, bool& zero) {
  __shared__ double red[8];
  __shared__ int bad;
  const int tid = threadIdx.x, nt = blockDim.x;
  if (tid == 0) bad = 0;
  double tr = 0.0;
  for (int i = tid; i < w; i += nt) tr += Gs[i * kL + i];
  tr = block_sum(tr, red);
  for (int t = tid; t < kW * kW; t += nt) {
    Rs[(t >> 6) * kL + (t & 63)] = 0.0;
    Xs[(t >> 6) * kL + (t & 63)] = 0.0;
  }
  zero = (tr == 0.0);
  if (zero) {
    __syncthreads();
    for (int i = tid; i < w; i += nt) {
      Rs[i * kL + i] = 1.0;
      Xs[i * kL + i] = 1.0;
    }
    __syncthreads();
    return true;
  }
  if (shift_coef > 0.0) {
    for (int i = tid; i < w; i += nt) Gs[i * kL + i] += shift_coef * tr;
  }
  __syncthreads();
  const int tx = tid & 63, ty = tid >> 6, nty = nt >> 6;
  for (int j = 0; j < w; ++j) {
    double d = Gs[j * kL + j];
    if (!(d > 0.0) || !isfinite(d)) {
      if (tid == 0) bad = 1;
      d = d > 0.0 ? d : 1e-300;
    }
    const double rjj = sqrt(d);
    if (ty == 0 && tx >= j && tx < w) Rs[j * kL + tx] = (tx == j) ? rjj : Gs[j * kL + tx] / rjj;
    __syncthreads();
    if (tx > j && tx < w) {
      const double rq = Rs[j * kL + tx];
      for (int k = j + 1 + ty; k <= tx; k += nty) Gs[k * kL + tx] -= Rs[j * kL + k] * rq;
    }
    __syncthreads();
  }
  // X = R^-1, rows from the bottom, 4 lanes per column
  const int c = tid >> 2, sub = tid & 3;
  for (int i = w - 1; i >= 0; --i) {
    double acc = 0.0;
    if (c < w && c >= i)
      for (int k = i + 1 + sub; k <= c; k += 4) acc = fma(Rs[i * kL + k], Xs[k * kL + c], acc);
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    acc += __shfl_xor_sync(0xffffffffu, acc, 2);
    if (c < w && c >= i && sub == 0) Xs[i * kL + c] = ((i == c ? 1.0 : 0.0) - acc) / Rs[i * kL + i];
    __syncthreads();
  }
  return bad == 0;
}

// out(rows x w) = in(rows x w) * Xs (upper triangular), chunk in smem (Cs),
// result written to global dst (ld ldd).  256 threads: thread -> (row, 16 cols).
FFB_DEV void apply_upper(const double* Cs, int rows, int w, const double* Xs, double* dst,
                         int64_t ldd, int64_t row0) {
  const int tid = threadIdx.x;
  for (int t = tid; t < rows * 4; t += blockDim.x) {
    const int r = t >> 2, cg = (t & 3) * 16;
    double acc[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) acc[q] = 0.0;
    for (int k = 0; k < w; ++k) {
      const double x = Cs[r * kL + k];
#pragma unroll
      for (int q = 0; q < 16; ++q) acc[q] = fma(x, Xs[k * kL + cg + q], acc[q]);
    }
#pragma unroll
    for (int q = 0; q < 16; ++q)
      if (cg + q < w) dst[(row0 + r) + (int64_t)(cg + q) * ldd] = acc[q];
  }
}

}  // namespace

__global__ void __launch_bounds__(256, 1) panel_qr_kernel(PanelArgs a) {
  extern __shared__ __align__(16) double sm[];
  double* Gs = sm;                    // w x w Gram / LU workspace
  double* Rs = Gs + kW * kL;          // Cholesky factor / L
  double* Xs = Rs + kW * kL;          // R^-1 / U
  double* Ra = Xs + kW * kL;          // Racc (every CTA keeps it; cheap)
  double* Cs = Ra + kW * kL;          // staged chunk of rows (kCH x w)
  double* Ws = Cs + kCH * kL;         // Ut / T staging
  __shared__ double Dd[kW];
  __shared__ int s_zero;
  const int tid = threadIdx.x, nt = blockDim.x, G = gridDim.x, w = a.w;
  const int64_t Mp = a.Mp;
  const int64_t r0 = (int64_t)blockIdx.x * a.rpc;
  const int64_t r1 = r0 + a.rpc < Mp ? r0 + a.rpc : Mp;
  const int ww = w * w;
  const int bi = (tid & 15) * 4, bj = (tid >> 4) * 4;
  bool zero = false;

  for (int pass = 0; pass < 3; ++pass) {
    const double* src = pass == 0 ? a.X : (pass == 1 ? a.Qa : a.Qb);
    const int64_t lds = pass == 0 ? a.ldx : Mp;
    double* dst = pass == 1 ? a.Qb : a.Qa;
    // (a) local Gram of rows [r0, r1)
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    for (int64_t c0 = r0; c0 < r1; c0 += kCH) {
      const int rows = (int)(r1 - c0 < kCH ? r1 - c0 : kCH);
      __syncthreads();
      for (int t = tid; t < rows * w; t += nt) {
        const int r = t % rows, c = t / rows;
        Cs[r * kL + c] = src[(c0 + r) + (int64_t)c * lds];
      }
      __syncthreads();
      for (int r = 0; r < rows; ++r) {
        double x[4], y[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          x[i] = Cs[r * kL + bi + i];
          y[i] = Cs[r * kL + bj + i];
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fma(x[i], y[j], acc[i][j]);
      }
    }
    double* mypart = a.part + (size_t)blockIdx.x * ww;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (bi + i < w && bj + j < w) mypart[(bi + i) + (bj + j) * w] = acc[i][j];
    grid_sync(a.bar, G);
    // (b) distributed fixed-order reduction
    {
      const int per = (ww + G - 1) / G;
      const int e0 = blockIdx.x * per, e1 = e0 + per < ww ? e0 + per : ww;
      for (int e = e0 + tid; e < e1; e += nt) {
        double s = 0.0;
        for (int c = 0; c < G; ++c) s += a.part[(size_t)c * ww + e];
        a.Gg[e] = s;
      }
    }
    grid_sync(a.bar, G);
    // (c) Cholesky + inverse (redundant in every CTA), Racc update
    for (int t = tid; t < ww; t += nt) {
      const int i = t % w, j = t / w;
      Gs[i * kL + j] = a.Gg[t];
    }
    __syncthreads();
    const double shift = pass == 0 ? 11.0 * ((double)Mp * w + (double)w * (w + 1)) * 1.1102230246251565e-16 : 0.0;
    bool zp = false;
    const bool ok = chol_inv(Gs, Rs, Xs, w, shift, zp);
    if (pass == 0) zero = zp;
    if (!ok && blockIdx.x == 0 && tid == 0) atomicOr(a.status, 2u /* kStCholFail */);
    // Racc <- R * Racc (pass 0: Racc = R; zero panel: Racc = 0)
    for (int t = tid; t < ww; t += nt) {
      const int i = t % w, j = t / w;
      double v = 0.0;
      if (zero) {
        v = 0.0;
      } else if (pass == 0) {
        v = Rs[i * kL + j];
      } else if (i <= j) {
        for (int k = i; k <= j; ++k) v = fma(Rs[i * kL + k], Ra[k * kL + j], v);
      }
      Gs[i * kL + j] = v;
    }
    __syncthreads();
    for (int t = tid; t < ww; t += nt) {
      const int i = t % w, j = t / w;
      Ra[i * kL + j] = Gs[i * kL + j];
    }
    // (d) own rows <- rows * R^-1
    for (int64_t c0 = r0; c0 < r1; c0 += kCH) {
      const int rows = (int)(r1 - c0 < kCH ? r1 - c0 : kCH);
      __syncthreads();
      for (int t = tid; t < rows * w; t += nt) {
        const int r = t % rows, c = t / rows;
        Cs[r * kL + c] = src[(c0 + r) + (int64_t)c * lds];
      }
      __syncthreads();
      apply_upper(Cs, rows, w, Xs, dst, Mp, c0);
    }
  }
  grid_sync(a.bar, G);   // Q = Qa complete (top w rows visible to every CTA)

  // (e) sign-fixing LU of Q_top * D - I (redundant in every CTA)
  if (tid == 0) s_zero = zero ? 1 : 0;
  double* q = Gs;   // w x w working copy of Q_top
  double* L = Rs;
  double* U = Xs;
  for (int t = tid; t < kW * kW; t += nt) {
    const int i = t >> 6, j = t & 63;
    q[i * kL + j] = (i < w && j < w) ? a.Qa[i + (int64_t)j * Mp] : 0.0;
    L[i * kL + j] = (i == j) ? 1.0 : 0.0;
    U[i * kL + j] = 0.0;
  }
  __syncthreads();
  if (!s_zero) {
    for (int c = 0; c < w; ++c) {
      const double z = q[c * kL + c];
      double d;
      if (fabs(z) == 1.0) d = z > 0.0 ? 1.0 : -1.0;   // identity reflector (tail == 0)
      else d = z > 0.0 ? -1.0 : 1.0;                  // pivot -(1+|z|) = -tau
      const double ucc = d * z - 1.0;
      if (tid == 0) {
        Dd[c] = d;
        U[c * kL + c] = ucc;
      }
      for (int i = c + 1 + tid; i < w; i += nt) L[i * kL + c] = ucc != 0.0 ? d * q[i * kL + c] / ucc : 0.0;
      for (int k = tid; k < c; k += nt) U[k * kL + c] = d * q[k * kL + c];
      __syncthreads();
      const int tx = tid & 63, ty = tid >> 6, nty = nt >> 6;
      if (tx > c && tx < w) {
        const double qc = q[c * kL + tx];
        for (int i = c + 1 + ty; i < w; i += nty) q[i * kL + tx] -= L[i * kL + c] * qc;
      }
      __syncthreads();
    }
  } else {
    for (int i = tid; i < w; i += nt) Dd[i] = 1.0;
    __syncthreads();
  }
  // Ui = D * U^{-1} (into Cs, zero-pivot rule) and T = -U L^{-T} (into Ws)
  double* Ui = Cs;
  double* Ts = Ws;
  {
    const int i = tid >> 2, sub = tid & 3;
    for (int c = 0; c < w; ++c) {
      double a0 = 0.0, a1 = 0.0;
      if (i < w)
        for (int k = sub; k < c; k += 4) {
          a0 = fma(Ui[i * kL + k], U[k * kL + c], a0);
          a1 = fma(Ts[i * kL + k], L[c * kL + k], a1);
        }
      a0 += __shfl_xor_sync(0xffffffffu, a0, 1);
      a0 += __shfl_xor_sync(0xffffffffu, a0, 2);
      a1 += __shfl_xor_sync(0xffffffffu, a1, 1);
      a1 += __shfl_xor_sync(0xffffffffu, a1, 2);
      if (i < w && sub == 0) {
        const double ucc = U[c * kL + c];
        Ui[i * kL + c] = (ucc != 0.0 && !s_zero) ? ((i == c ? 1.0 : 0.0) - a0) / ucc : 0.0;
        Ts[i * kL + c] = s_zero ? 0.0 : -U[i * kL + c] - a1;
      }
      __syncthreads();
    }
  }
  // scale rows of Ui by D (Y2 = Q_bottom * D * U^-1)
  for (int t = tid; t < ww; t += nt) {
    const int i = t % w, j = t / w;
    Ui[i * kL + j] *= Dd[i];
  }
  __syncthreads();
  if (blockIdx.x == 0) {
    for (int t = tid; t < ww; t += nt) {
      const int i = t % w, j = t / w;
      a.Y[i + (int64_t)j * a.ldy] = L[i * kL + j];
      a.T[i + (int64_t)j * a.ldt] = Ts[i * kL + j];
      a.R[i + (int64_t)j * a.ldr] = (i <= j) ? Dd[i] * Ra[i * kL + j] : 0.0;
    }
  }
  // (f) Y rows >= w: Y = Q * (D U^-1)  (Ui is upper triangular)
  {
    const int64_t y0 = r0 > w ? r0 : w;
    // Ws is reused as the row stage (Ts no longer needed after CTA 0 wrote it)
    __syncthreads();
    double* Ys = Ws;
    for (int64_t c0 = y0; c0 < r1; c0 += kCH) {
      const int rows = (int)(r1 - c0 < kCH ? r1 - c0 : kCH);
      __syncthreads();
      for (int t = tid; t < rows * w; t += nt) {
        const int r = t % rows, c = t / rows;
        Ys[r * kL + c] = a.Qa[(c0 + r) + (int64_t)c * Mp];
      }
      __syncthreads();
      apply_upper(Ys, rows, w, Ui, a.Y, a.ldy, c0);
    }
  }
}

size_t panel_smem_bytes() { return sizeof(double) * (size_t)(5 * kW * kL + kCH * kL); }

int panel_grid(int sms, int64_t Mp) {
  int64_t g = (Mp + 63) / 64;
  if (g > sms) g = sms;
  if (g < 1) g = 1;
  return (int)g;
}

cudaError_t launch_panel_qr(cudaStream_t st, int sms, const double* X, int64_t ldx, int64_t Mp,
                            int w, double* Y, int64_t ldy, double* T, int64_t ldt, double* R,
                            int64_t ldr, double* Qa, double* Qb, double* part, double* Gg,
                            uint32_t* bar, uint32_t* status) {
  static bool attr = false;
  const size_t smem = panel_smem_bytes();
  if (!attr) {
    cudaFuncSetAttribute(panel_qr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  const int G = panel_grid(sms, Mp);
  PanelArgs a{X, ldx, Mp, w, Y, ldy, T, ldt, R, ldr, Qa, Qb, part, Gg, bar, status,
              (int)((Mp + G - 1) / G)};
  cudaError_t e = cudaMemsetAsync(bar, 0, 2 * sizeof(uint32_t), st);
  if (e != cudaSuccess) return e;
  void* args[] = {&a};
  return cudaLaunchCooperativeKernel((void*)panel_qr_kernel, dim3(G), dim3(256), args, smem, st);
}

}  // namespace ffb
