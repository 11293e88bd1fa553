#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace ffb {

struct PanelArgs {
  const double* X;
  int64_t ldx;
  int64_t Mp;
  int w;
  double* Y;
  int64_t ldy;
  double* T;
  int64_t ldt;
  double* R;
  int64_t ldr;
  double* Qa;      // Mp x w work (ld Mp)
  double* Qb;      // Mp x w work (ld Mp)
  double* part;    // grid x w*w partial Grams
  double* Gg;      // w*w reduced Gram
  uint32_t* bar;   // [2] grid barrier
  uint32_t* status;
  int rpc;         // rows per CTA (Householder fallback)
  int vg;          // row groups of the CholeskyQR passes (fixed by Mp, not by the grid)
  int64_t gpr;     // rows per group
  long long* prof; // optional [8] phase cycles of CTA 0 (FFB_PANEL_PROF)
};

size_t panel_smem_bytes();
int panel_grid(int sms, int64_t Mp);

// Householder QR of one panel X (Mp x w, w <= 64): Y (Mp x w, unit lower
// trapezoidal), T (w x w upper), R (w x w upper) with the reference's signs.
cudaError_t launch_panel_qr(cudaStream_t st, int sms, const double* X, int64_t ldx, int64_t Mp,
                            int w, double* Y, int64_t ldy, double* T, int64_t ldt, double* R,
                            int64_t ldr, double* Qa, double* Qb, double* part, double* Gg,
                            uint32_t* bar, uint32_t* status);

}  // namespace ffb
