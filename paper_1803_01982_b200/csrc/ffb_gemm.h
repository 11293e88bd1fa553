#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace ffb {

struct GemmCtx {
  int sms = 148;
  double* partial = nullptr;   // split-K scratch
  size_t partial_cap = 0;      // doubles
  unsigned* counters = nullptr;  // stream-K per-tile arrival counters (zeroed)
  size_t counter_cap = 0;
  int64_t flops = 0;
  int64_t launches = 0;
};

// When non-null, the GEMM writes raw split-K partial tiles (ld = M) and does NOT
// reduce; used for Gram matrices that a single-CTA consumer reduces itself.
struct GemmPartialOut {
  int max_splits;
  double* part;
  int splits;
};

cudaError_t gemm_f64(GemmCtx& c, cudaStream_t st, int64_t M, int64_t N, int64_t K, double alpha,
                     const double* A, int64_t lda, bool akc, const double* B, int64_t ldb, bool bkc,
                     double beta, double* C, int64_t ldc, GemmPartialOut* pout = nullptr);

}  // namespace ffb
