#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace ffb {

struct JacobiArgs {
  double* M;
  int64_t ldm;
  double* V;
  int64_t ldv;
  int l, bs, nb;
  double tol;
  int max_sweeps;
  uint32_t* bar;     // [2] grid barrier
  double* offmax;    // [max_sweeps]
  int* sweeps;       // sweeps executed
  int inner;         // passes over the cross-block pairs per visit
  long long* prof;   // optional phase timers (debug)
};

int jacobi_block_size(int l);

// SVD of the l x l matrix M (overwritten): sorted sig (l), U (l x l) and V (l x l)
// with M = U diag(sig) V^T.  V must be initialised to the identity by the caller.
cudaError_t launch_jacobi_svd(cudaStream_t st, int sms, double* M, int64_t ldm, double* V,
                              int64_t ldv, int l, double* sig, double* U, int64_t ldu, double* Vo,
                              int64_t ldvo, uint32_t* bar, double* offmax, int* sweeps, int* order,
                              int max_sweeps);

}  // namespace ffb
