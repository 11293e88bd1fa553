#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace ffb {

struct JacobiArgs {
  double* M;         // lpad x ncp row-major (padded, zero filled)
  double* jhist;     // [max_sweeps][nb - 1][nb / 2][32 x 32] recorded rotations
  int64_t ld;        // = ncp
  int l, lpad, nb;
  double tol;
  int max_sweeps;
  uint32_t* bar;     // [2] grid barrier
  double* offmax;    // [max_sweeps]
  int* sweeps;       // [0] sweeps executed, [1] prescale exponent
  int inner;         // passes over the cross-block pairs per visit
  long long* prof;   // optional phase timers (debug)
  int P;             // Jacobi CTAs (block pairs); CTAs >= P replay V (fused launch)
  double* V;         // lpad x ncp row-major V (written by the replay)
  uint32_t* progress;  // [0] rounds published, [1] total rounds + 1 when done
  int fused;
  double* gdiag;     // [nb][kBS x kBS] diagonal Gram blocks carried between rounds
  int lean;          // rotation formula: 1 = two-MUFU hypot form, 0 = zeta / Newton form
};

int jacobi_block_size(int l);
size_t jacobi_work_doubles(int l, int max_sweeps);

// SVD of the l x l column-major matrix M (read only): sorted sig (l), U (l x l)
// and Vo (l x l) with M = U diag(sig) Vo^T.  work: jacobi_work_doubles(l).
cudaError_t launch_jacobi_svd(cudaStream_t st, int sms, const double* M, int64_t ldm, int l,
                              double* sig, double* U, int64_t ldu, double* Vo, int64_t ldvo,
                              double* work, uint32_t* bar, double* offmax, int* sweeps, int* order,
                              int max_sweeps);

// Column-ring variant (ffb_jacobi_ring.cu) for small l: whole iterate in one
// cluster's distributed shared memory.  Same contract as launch_jacobi_svd;
// work needs jacobi_work_doubles(l) (it uses less).
bool jacobi_ring_supported(int l, int sms);
cudaError_t launch_jacobi_ring(cudaStream_t st, int sms, const double* M, int64_t ldm, int l,
                               double* sig, double* U, int64_t ldu, double* Vo, int64_t ldvo,
                               double* work, double* offmax, int* sweeps, int* order,
                               int max_sweeps);
// sweeps[1] <- exponent e with 2^e ~ max |M| (the power-of-two prescale)
cudaError_t launch_jacobi_scale(cudaStream_t st, const double* M, int64_t ldm, int l, int* sweeps);

}  // namespace ffb
