// Launch interfaces of the non-GEMM kernels (definitions in ffb_kernels.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace ffb {

// Device status word bits (OR-ed by kernels, read by the host at sync points).
enum : uint32_t {
  kStNonFinite = 1u << 0,       // NaN/Inf in the input or a factor
  kStCholFail = 1u << 1,        // Cholesky of a panel Gram broke down
  kStSingular = 1u << 2,        // zero diagonal in Rtilde (g2 solve)
  kStZeroPivot = 1u << 3,       // exact zero on a TRQRCP R11 diagonal (sketch update)
};

struct PivotArgs {
  const double* B;
  int64_t ldb;
  int s;
  int64_t n;
  int64_t j0;
  int bb;
  int64_t* arr;
  int64_t* pos;
  int G;
  int cpc;
  int sP;              // padded per-column stride (set by launch_pivots)
  double* work;        // !smem mode: G * sP * cpc
  unsigned long long* rec;  // [2][G][recw] tagged exchange records, zero on entry
  int recw;            // words per record (pivots_recw(s))
  int64_t* hist;       // [bb] winning positions
  double* gap;         // [bb] relative top-2 gap per step (certified near-tie evidence)
  long long* prof;     // optional [G][8] phase cycle sums (FFB_PIV_PROF)
};

// Scalars block shared between SRQR kernels and the host (device memory).
struct SrqrScalars {
  double alpha;
  double anorm;
  double g2;
  double g1;
  double r22;
  double tau;
  double tau_hat;
  double spare;
  int64_t i_off;
  int64_t piv;
  uint32_t status;
  uint32_t need_swap;
};

cudaError_t launch_colsq(cudaStream_t st, const double* A, int64_t lda, int64_t m, int64_t n,
                         double* colsq);
size_t colsq_rm_part_doubles(int64_t n);
cudaError_t launch_colsq_rm(cudaStream_t st, const double* A, int64_t lda, int64_t m, int64_t n,
                            double* part, double* colsq);
cudaError_t launch_gather_cols_strided(cudaStream_t st, const double* src, int64_t rs, int64_t cs,
                                       int64_t rows, const int64_t* idx, int64_t ncols, double* dst,
                                       int64_t ld_dst);
cudaError_t launch_copy_rows_rm(cudaStream_t st, const double* src, int64_t ld_src, int64_t rows,
                                int64_t cols, double* dst, int64_t ld_dst);
cudaError_t launch_iota2(cudaStream_t st, int64_t* arr, int64_t* pos, int64_t n);
cudaError_t launch_pivots(cudaStream_t st, const PivotArgs& a, bool smem_mode, size_t smem);
size_t pivots_smem_bytes(int s, int cpc, bool smem_mode);
int pivots_stride(int s);
int pivots_recw(int s);
void* pivots_kernel_ptr(bool smem_mode, int rq, int s);
int pivots_rq(int s, int cpc, bool smem_mode);

cudaError_t launch_gather_cols(cudaStream_t st, const double* src, int64_t ld_src, int64_t rows,
                               const int64_t* idx, int64_t ncols, double* dst, int64_t ld_dst);
cudaError_t launch_scatter_rows(cudaStream_t st, const double* src, int64_t ld_src, int64_t nrows,
                                int64_t ncols, const int64_t* idx, double* dst, int64_t ld_dst);
cudaError_t launch_copy_bytes(cudaStream_t st, const void* src, void* dst, size_t bytes);
cudaError_t launch_copy_rows(cudaStream_t st, const double* src, int64_t ld_src, int64_t rows,
                             int64_t cols, double* dst, int64_t ld_dst);
cudaError_t launch_fill(cudaStream_t st, double* p, size_t count, double v);
cudaError_t launch_add_identity(cudaStream_t st, double* X, int64_t ld, int64_t rows,
                                int64_t cols, double scale);
cudaError_t launch_add_top(cudaStream_t st, double* X, int64_t ldx, const double* Y, int64_t ldy,
                           int64_t rows, int64_t cols);

// Panel reconstruction pieces.
cudaError_t launch_cholinv(cudaStream_t st, const double* G, int w, int64_t rows_m, bool shift,
                           bool first, double* Racc, double* Rinv, uint32_t* status);
cudaError_t launch_signlu(cudaStream_t st, const double* Qtop, int64_t ldq, int w,
                          const double* Racc, double* Y, int64_t ldy, double* T, int64_t ldt,
                          double* R, int64_t ldr, double* Ut, double* D);

// TRQRCP helpers.
cudaError_t launch_fix_rrows(cudaStream_t st, double* R, int64_t ldr, int64_t j0, int bb,
                             const int64_t* arr, const double* Rb, int64_t ldrb);
cudaError_t launch_triinv_upper(cudaStream_t st, const double* Rb, int64_t ldrb, int w,
                                double* Rinv, int64_t ldo, uint32_t* status);

// SRQR.
cudaError_t launch_rinit(cudaStream_t st, const double* B, int64_t ldb, int s, const int64_t* arr,
                         int64_t n, int64_t l, double* r, double* rinit);
cudaError_t launch_anorm(cudaStream_t st, const double* colsq, int64_t n, SrqrScalars* sc);
cudaError_t launch_ext_pick(cudaStream_t st, int64_t l, int64_t n, int64_t* arr, int64_t* pos,
                            double* r, double* rinit, SrqrScalars* sc);
cudaError_t launch_ext_project(cudaStream_t st, const double* A, int64_t ars, int64_t acs, int64_t m, int64_t l,
                               const double* Q, int64_t ldq, const double* R, int64_t ldr,
                               const int64_t* arr, double* u, double* ct, double* part,
                               SrqrScalars* sc, double* r, double* Rfull);
cudaError_t launch_ext_row(cudaStream_t st, const double* A, int64_t ars, int64_t acs, int64_t m, int64_t n,
                           int64_t l, const double* Q, int64_t ldq, double* R, int64_t ldr,
                           const int64_t* arr, const double* colsq, double* r,
                           const double* rinit, const SrqrScalars* sc);
cudaError_t launch_ext_finish(cudaStream_t st, const double* part, int nparts, int64_t l, int64_t n,
                              const int64_t* arr, double* R, int64_t ldr, double* r,
                              SrqrScalars* sc, const double* u, int64_t m, double* Ql);
cudaError_t launch_g2(cudaStream_t st, const double* R, int64_t ldr, const int64_t* arr, int64_t l,
                      const double* omega, int d, double g, double* Z, SrqrScalars* sc);
cudaError_t launch_g2big_prep(cudaStream_t st, double* Rt, int64_t L1, const double* omega, int d,
                              double* Z, const SrqrScalars* sc, uint32_t* flag);
cudaError_t launch_g2big_diag(cudaStream_t st, const double* Rt, int64_t L1, int64_t i0, int nbk,
                              double* Z, int d);
cudaError_t launch_g2big_finish(cudaStream_t st, const double* Z, int64_t L1, int d, double g,
                                const uint32_t* flag, SrqrScalars* sc);
cudaError_t launch_pack(cudaStream_t st, const double* R, int64_t ldr, const int64_t* arr,
                        const double* colsq, int64_t l, int64_t n, double* part, int64_t swaps,
                        SrqrScalars* sc);
cudaError_t launch_rotate_out(cudaStream_t st, double* R, int64_t ldr, double* Q, int64_t ldq,
                              int64_t m, int64_t n, int64_t l, int64_t* arr, int64_t* pos,
                              double* r, double* rinit, const SrqrScalars* sc, double* rot);
cudaError_t launch_revert(cudaStream_t st, const double* R, int64_t ldr, const int64_t* arr,
                          int64_t l, int64_t n, double* r);

// Outputs.
cudaError_t launch_r_arranged(cudaStream_t st, const double* R, int64_t ldr, const int64_t* arr,
                              int64_t rows, int64_t n, double* out, int64_t ldo,
                              int64_t tri_rows);
cudaError_t launch_build_rt(cudaStream_t st, const double* R, int64_t ldr, const int64_t* arr,
                            int64_t l, int64_t n, double* X, int64_t ldx);
cudaError_t launch_diag(cudaStream_t st, const double* R, int64_t ldr, int64_t nd, double* out);
cudaError_t launch_finite_check(cudaStream_t st, const double* x, size_t count, uint32_t* status);

}  // namespace ffb
